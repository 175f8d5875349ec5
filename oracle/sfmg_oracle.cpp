/*
 * sfmg_oracle.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, deliberately unoptimised CPU reference for what the B200 hot path
 * (paper_1402_5938_b200/csrc) computes: the LGL tensor basis, the structured hex mesh and
 * its numbering, isoparametric geometric factors, the variable-coefficient stiffness operator
 * -div(mu grad u), its diagonal, the power-iteration lambda_max estimate, the Chebyshev-
 * accelerated Jacobi smoother, p-prolongation/restriction, the p-multigrid V-cycle and the
 * MG solver / MG-preconditioned CG of Algorithm 1.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
 * may load this library.  It shares no code, header, table or constant generator with the
 * CUDA path; the two only share the seeded *input* generator (paper_1402_5938_b200/inputs.py),
 * and the power-iteration start vector, which each side draws from its own copy of the same
 * counter-based splitmix64 generator (reading R9/R15).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (arXiv 1402.5938), "S:n" = SPEC.md line
 * n, "R<k>" = reading k in DESIGN.md section 3 (the paper is silent or ambiguous there).
 *
 * Tiers:
 *   O1  dense element matrices by direct quadrature (orc_element_matrix, orc_assemble_dense)
 *   O2  unassembled direct quadrature: every basis gradient tabulated per (node, point)
 *       pair, no tensor or collocation structure used (orc_apply with tier=2)
 *   O3  plain sum-factorised loops (tier=3), pinned against O1/O2 by tests, used only where
 *       O2 is too slow (iterative solves at config-5 size)
 * Geometry tiers: dense definition J = sum_l x_l (grad phi_l)^T  (geom_tier=2) and the
 * factorised form that uses the collocation property ell_a(xhat_i)=delta_ai (geom_tier=3),
 * pinned against each other by tests.
 *
 * Build: g++ -O2 -ffp-contract=off -fopenmp -shared -fPIC (R23: no FMA contraction).
 * Determinism: every scatter runs colour by colour (8 element colours); within a colour
 * no two elements share a node, so results do not depend on the thread count.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <vector>
#include <omp.h>

namespace {

const double kPi = 3.14159265358979323846;

/* ------------------------------------------------------------------ 1-D basis */

// Legendre P_p(x) and P_p'(x) by the three-term recurrence (Bonnet).
void legendre(int p, double x, double* P, double* dP) {
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
  if (p == 0) { *P = 1.0; *dP = 0.0; return; }
  for (int k = 1; k < p; ++k) {
    double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
    double d2 = d0 + (2.0 * k + 1.0) * p1;   // P'_{k+1} = P'_{k-1} + (2k+1) P_k
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  *P = p1; *dP = d1;
}

// LGL nodes: -1, the p-1 roots of P_p', +1; weights 2/(p(p+1) P_p(x_i)^2).
// Newton on P_p' from Chebyshev-Gauss-Lobatto guesses, P'' from the Legendre ODE
// (1-x^2) P'' = 2x P' - p(p+1) P; then symmetrised.
void lgl(int p, std::vector<double>& x, std::vector<double>& w) {
  int n = p + 1;
  x.assign(n, 0.0); w.assign(n, 0.0);
  x[0] = -1.0; x[p] = 1.0;
  for (int i = 1; i < p; ++i) {
    double xi = -std::cos(kPi * i / p);
    for (int it = 0; it < 200; ++it) {
      double P, dP;
      legendre(p, xi, &P, &dP);
      double d2P = (2.0 * xi * dP - p * (p + 1.0) * P) / (1.0 - xi * xi);
      double dx = dP / d2P;
      xi -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < n / 2; ++i) {       // symmetrise: x_{p-i} = -x_i, centre exactly 0
    double a = 0.5 * (x[p - i] - x[i]);
    x[i] = -a; x[p - i] = a;
  }
  if (p % 2 == 0) x[p / 2] = 0.0;
  for (int i = 0; i < n; ++i) {
    double P, dP;
    legendre(p, x[i], &P, &dP);
    w[i] = 2.0 / (p * (p + 1.0) * P * P);
  }
}

// Lagrange cardinal polynomial ell_m on nodes xs, and its derivative (product rule).
double lagrange(const std::vector<double>& xs, int m, double t) {
  double v = 1.0;
  for (size_t k = 0; k < xs.size(); ++k)
    if ((int)k != m) v *= (t - xs[k]) / (xs[m] - xs[k]);
  return v;
}
double dlagrange(const std::vector<double>& xs, int m, double t) {
  double s = 0.0;
  for (size_t j = 0; j < xs.size(); ++j) {
    if ((int)j == m) continue;
    double prod = 1.0 / (xs[m] - xs[j]);
    for (size_t k = 0; k < xs.size(); ++k)
      if ((int)k != m && k != j) prod *= (t - xs[k]) / (xs[m] - xs[k]);
    s += prod;
  }
  return s;
}

// Gauss-Legendre points (roots of P_n) and weights 2 / ((1 - x^2) P_n'(x)^2), by Newton from
// cos(pi (i + 3/4) / (n + 1/2)).  NEXT-3 ("Gauss quadrature").
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0); w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = -std::cos(kPi * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre(n, t, &P, &dP);
      double dt = P / dP;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    double P, dP;
    legendre(n, t, &P, &dP);
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * dP * dP);
  }
  for (int i = 0; i < n / 2; ++i) {   // symmetrise
    double a = 0.5 * (x[n - 1 - i] - x[i]);
    x[i] = -a; x[n - 1 - i] = a;
    double ww = 0.5 * (w[i] + w[n - 1 - i]);
    w[i] = w[n - 1 - i] = ww;
  }
  if (n % 2) x[n / 2] = 0.0;
}

struct Basis {
  int p = 0, n = 0;
  int quad = 0;             // 0: LGL points collocated with the nodes (R1); 1: n Gauss-Legendre points (NEXT-3)
  std::vector<double> x, w;  // LGL nodes / weights
  std::vector<double> qx, qw;   // quadrature points / weights
  std::vector<double> L;   // L[i*n+a]  = ell_a(q_i)   (tabulated, no delta shortcut)
  std::vector<double> dL;  // dL[i*n+a] = ell_a'(q_i)  (the D matrix when collocated)
  void build(int p_, int quad_ = 0) {
    p = p_; n = p + 1; quad = quad_;
    lgl(p, x, w);
    if (quad == 1) gauss_legendre(n, qx, qw);
    else { qx = x; qw = w; }
    L.assign(n * n, 0.0); dL.assign(n * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < n; ++a) {
        L[i * n + a] = lagrange(x, a, qx[i]);
        dL[i * n + a] = dlagrange(x, a, qx[i]);
      }
  }
};
static int g_quad = 0;   // quadrature of levels created from now on (orc_set_quadrature)

/* ------------------------------------------------------------------ seeded generator (R9, R15) */

inline uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline double uniform_pm1(uint64_t seed, uint64_t i) {
  return 2.0 * ((double)(splitmix64_at(seed, i) >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

/* ------------------------------------------------------------------ coefficient mu (R3, R6) */

// kind 0: c0; 1: exp(c1 S); 2: 10^(c1 S); 3: c0 + c1 sum_i cos^2(2 pi x_i) (paper 3d-var form);
// 100 (oracle-only, used by the separable pin): exp(c1 (x + 2y + 3z)).  S = sin2pix sin2piy sin2piz.
double coeff_mu(int kind, double c0, double c1, double x, double y, double z) {
  double S = std::sin(2 * kPi * x) * std::sin(2 * kPi * y) * std::sin(2 * kPi * z);
  switch (kind) {
    case 0: return c0;
    case 1: return std::exp(c1 * S);
    case 2: return std::pow(10.0, c1 * S);
    case 3: {
      double a = std::cos(2 * kPi * x), b = std::cos(2 * kPi * y), c = std::cos(2 * kPi * z);
      return c0 + c1 * (a * a + b * b + c * c);
    }
    case 100: return std::exp(c1 * x) * std::exp(2.0 * c1 * y) * std::exp(3.0 * c1 * z);
  }
  return NAN;
}
void coeff_grad(int kind, double c0, double c1, double x, double y, double z, double g[3]) {
  double sx = std::sin(2 * kPi * x), sy = std::sin(2 * kPi * y), sz = std::sin(2 * kPi * z);
  double cx = std::cos(2 * kPi * x), cy = std::cos(2 * kPi * y), cz = std::cos(2 * kPi * z);
  double dS[3] = {2 * kPi * cx * sy * sz, 2 * kPi * sx * cy * sz, 2 * kPi * sx * sy * cz};
  double mu = coeff_mu(kind, c0, c1, x, y, z);
  switch (kind) {
    case 0: g[0] = g[1] = g[2] = 0; return;
    case 1: for (int d = 0; d < 3; ++d) g[d] = c1 * mu * dS[d]; return;
    case 2: for (int d = 0; d < 3; ++d) g[d] = std::log(10.0) * c1 * mu * dS[d]; return;
    case 3: {
      double xs[3] = {x, y, z};
      for (int d = 0; d < 3; ++d) g[d] = -2 * kPi * c1 * std::sin(4 * kPi * xs[d]);
      return;
    }
    case 100: g[0] = c1 * mu; g[1] = 2 * c1 * mu; g[2] = 3 * c1 * mu; return;
  }
}

/* ------------------------------------------------------------------ level: mesh + geometry */

struct Level {
  int nex, ney, nez, p, n, warp, coeff;
  double amp, c0, c1;
  int64_t E, N, Mx, My, Mz, n3;
  int geom_tier;            // 2 dense definition, 3 factorised
  int tier;                 // apply tier: 2 (O2) or 3 (O3)
  bool eager;
  Basis B;
  std::vector<double> G;    // [E][6][n3] when eager
  std::vector<double> detJ; // [E][n3] when eager
  std::vector<double> diag_cache;  // diag(A_D), computed on first use
  std::vector<int64_t> gslot;      // lazy mode: element -> slot in Gcache (-1: not cached)
  std::vector<double> Gcache;      // [slots][6][n3]
  double min_detj = 1e300;
  int status = 0;           // 0 ok, 4 geometry (det J <= 0)
  std::vector<std::vector<int64_t>> colour_elems;

  void elem_coords(int64_t e, int& ex, int& ey, int& ez) const {
    ex = (int)(e % nex); ey = (int)((e / nex) % ney); ez = (int)(e / ((int64_t)nex * ney));
  }
  // lattice numbering (pinned against orc_l2g_by_matching by tests)
  int64_t gidx(int64_t I, int64_t J, int64_t K) const { return I + Mx * (J + My * K); }
  int64_t l2g(int64_t e, int a, int b, int c) const {
    int ex, ey, ez; elem_coords(e, ex, ey, ez);
    return gidx((int64_t)ex * p + a, (int64_t)ey * p + b, (int64_t)ez * p + c);
  }
  bool boundary(int64_t g) const {
    int64_t I = g % Mx, J = (g / Mx) % My, K = g / (Mx * My);
    return I == 0 || I == Mx - 1 || J == 0 || J == My - 1 || K == 0 || K == Mz - 1;
  }
};

// Physical node coordinates of element e: reference-cube point X then the warp (R5).
void element_nodes(const Level& L, int64_t e, std::vector<double>& X) {
  int n = L.n; int64_t n3 = L.n3;
  X.assign(3 * n3, 0.0);
  int ex, ey, ez; L.elem_coords(e, ex, ey, ez);
  for (int c = 0; c < n; ++c)
    for (int b = 0; b < n; ++b)
      for (int a = 0; a < n; ++a) {
        int64_t l = a + n * (b + n * c);
        double Xr = (ex + 0.5 * (L.B.x[a] + 1.0)) / L.nex;
        double Yr = (ey + 0.5 * (L.B.x[b] + 1.0)) / L.ney;
        double Zr = (ez + 0.5 * (L.B.x[c] + 1.0)) / L.nez;
        double s = 0.0;
        if (L.warp == 1) s = L.amp * std::sin(kPi * Xr) * std::sin(kPi * Yr) * std::sin(kPi * Zr);
        X[l] = Xr + s; X[n3 + l] = Yr + s; X[2 * n3 + l] = Zr + s;
      }
}

// grad_ref phi_l at quadrature point q, from 1-D tabulations (no delta shortcut).
inline void grad_phi(const Basis& B, int i, int j, int k, int a, int b, int c, double d[3]) {
  int n = B.n;
  double La = B.L[i * n + a], Lb = B.L[j * n + b], Lc = B.L[k * n + c];
  double dLa = B.dL[i * n + a], dLb = B.dL[j * n + b], dLc = B.dL[k * n + c];
  d[0] = dLa * Lb * Lc; d[1] = La * dLb * Lc; d[2] = La * Lb * dLc;
}

// Physical position of quadrature point (i,j,k): x(xi_q) = sum_l x_l phi_l(xi_q) (isoparametric map).
inline void quad_point(const Level& L, const std::vector<double>& X, int i, int j, int k, double xq[3]) {
  int n = L.n; int64_t n3 = L.n3;
  xq[0] = xq[1] = xq[2] = 0.0;
  for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
    int64_t l = a + n * (b + n * c);
    double ph = L.B.L[i * n + a] * L.B.L[j * n + b] * L.B.L[k * n + c];
    xq[0] += ph * X[l]; xq[1] += ph * X[n3 + l]; xq[2] += ph * X[2 * n3 + l];
  }
}

// Isoparametric geometric factors of one element (R1, R2, R3):
// G_q = w_i w_j w_k mu(x_q) detJ_q J_q^{-1} J_q^{-T}, J[al][be] = d x_al / d xi_be.
// Returns min det J over the element.
double element_geometry(const Level& L, int64_t e, double* G, double* dJ, int geom_tier) {
  int n = L.n; int64_t n3 = L.n3;
  std::vector<double> X;
  element_nodes(L, e, X);
  double mind = 1e300;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int64_t q = i + n * (j + n * k);
        double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        if (geom_tier == 2) {
          for (int c = 0; c < n; ++c)
            for (int b = 0; b < n; ++b)
              for (int a = 0; a < n; ++a) {
                int64_t l = a + n * (b + n * c);
                double d[3];
                grad_phi(L.B, i, j, k, a, b, c, d);
                for (int al = 0; al < 3; ++al)
                  for (int be = 0; be < 3; ++be) J[al][be] += X[al * n3 + l] * d[be];
              }
        } else {
          for (int al = 0; al < 3; ++al)
            for (int m = 0; m < n; ++m) {
              J[al][0] += L.B.dL[i * n + m] * X[al * n3 + (m + n * (j + n * k))];
              J[al][1] += L.B.dL[j * n + m] * X[al * n3 + (i + n * (m + n * k))];
              J[al][2] += L.B.dL[k * n + m] * X[al * n3 + (i + n * (j + n * m))];
            }
        }
        double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
                   - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
                   + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        mind = std::min(mind, det);
        double Ji[3][3];   // inverse via adjugate
        Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
        Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
        Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
        Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
        Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
        Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
        Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
        Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
        Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
        double xq[3] = {X[q], X[n3 + q], X[2 * n3 + q]};   // collocated: the node itself
        if (L.B.quad == 1) quad_point(L, X, i, j, k, xq);
        double mu = coeff_mu(L.coeff, L.c0, L.c1, xq[0], xq[1], xq[2]);
        double s = L.B.qw[i] * L.B.qw[j] * L.B.qw[k] * mu * det;
        double M[3][3];
        for (int al = 0; al < 3; ++al)
          for (int be = 0; be < 3; ++be) {
            double t = 0.0;
            for (int ga = 0; ga < 3; ++ga) t += Ji[al][ga] * Ji[be][ga];
            M[al][be] = s * t;
          }
        G[0 * n3 + q] = M[0][0]; G[1 * n3 + q] = M[0][1]; G[2 * n3 + q] = M[0][2];
        G[3 * n3 + q] = M[1][1]; G[4 * n3 + q] = M[1][2]; G[5 * n3 + q] = M[2][2];
        if (dJ) dJ[q] = det;
      }
  return mind;
}

// Fetch G of element e: from the eager store, else computed into buf.
const double* elem_G(const Level& L, int64_t e, std::vector<double>& buf) {
  if (L.eager) return &L.G[(size_t)e * 6 * L.n3];
  if (!L.gslot.empty() && L.gslot[e] >= 0) return &L.Gcache[(size_t)L.gslot[e] * 6 * L.n3];
  buf.resize(6 * L.n3);
  element_geometry(L, e, buf.data(), nullptr, L.geom_tier);
  return buf.data();
}

/* ------------------------------------------------------------------ element operators */

// O2: v_l = sum_q grad phi_l(q)^T G_q sum_m u_m grad phi_m(q); dense tabulation, 6 n^6 FMA.
void element_apply_o2(const Level& L, const double* G, const double* u, double* v) {
  int n = L.n; int64_t n3 = L.n3;
  for (int64_t l = 0; l < n3; ++l) v[l] = 0.0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int64_t q = i + n * (j + n * k);
        double g[3] = {0, 0, 0};
        for (int c = 0; c < n; ++c)
          for (int b = 0; b < n; ++b)
            for (int a = 0; a < n; ++a) {
              int64_t m = a + n * (b + n * c);
              double d[3];
              grad_phi(L.B, i, j, k, a, b, c, d);
              g[0] += d[0] * u[m]; g[1] += d[1] * u[m]; g[2] += d[2] * u[m];
            }
        double w0 = G[0 * n3 + q] * g[0] + G[1 * n3 + q] * g[1] + G[2 * n3 + q] * g[2];
        double w1 = G[1 * n3 + q] * g[0] + G[3 * n3 + q] * g[1] + G[4 * n3 + q] * g[2];
        double w2 = G[2 * n3 + q] * g[0] + G[4 * n3 + q] * g[1] + G[5 * n3 + q] * g[2];
        for (int c = 0; c < n; ++c)
          for (int b = 0; b < n; ++b)
            for (int a = 0; a < n; ++a) {
              int64_t l = a + n * (b + n * c);
              double d[3];
              grad_phi(L.B, i, j, k, a, b, c, d);
              v[l] += d[0] * w0 + d[1] * w1 + d[2] * w2;
            }
      }
}

// O3: the same result by 1-D (sum-factorised) loops: grad = (D x I x I, I x D x I, I x I x D) u,
// w = G grad, v = D^T-contractions of w.
void element_apply_o3(const Level& L, const double* G, const double* u, double* v) {
  int n = L.n; int64_t n3 = L.n3;
  const std::vector<double>& D = L.B.dL;
  std::vector<double> w0(n3), w1(n3), w2(n3);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int64_t q = i + n * (j + n * k);
        double g0 = 0, g1 = 0, g2 = 0;
        for (int m = 0; m < n; ++m) {
          g0 += D[i * n + m] * u[m + n * (j + n * k)];
          g1 += D[j * n + m] * u[i + n * (m + n * k)];
          g2 += D[k * n + m] * u[i + n * (j + n * m)];
        }
        w0[q] = G[0 * n3 + q] * g0 + G[1 * n3 + q] * g1 + G[2 * n3 + q] * g2;
        w1[q] = G[1 * n3 + q] * g0 + G[3 * n3 + q] * g1 + G[4 * n3 + q] * g2;
        w2[q] = G[2 * n3 + q] * g0 + G[4 * n3 + q] * g1 + G[5 * n3 + q] * g2;
      }
  for (int c = 0; c < n; ++c)
    for (int b = 0; b < n; ++b)
      for (int a = 0; a < n; ++a) {
        double s = 0.0;
        for (int m = 0; m < n; ++m) {
          s += D[m * n + a] * w0[m + n * (b + n * c)];
          s += D[m * n + b] * w1[a + n * (m + n * c)];
          s += D[m * n + c] * w2[a + n * (b + n * m)];
        }
        v[a + n * (b + n * c)] = s;
      }
}

// O1: dense element matrix K[l][m] = sum_q grad phi_l(q)^T G_q grad phi_m(q).
void element_matrix(const Level& L, const double* G, double* K) {
  int n = L.n; int64_t n3 = L.n3;
  std::vector<double> T(3 * n3 * n3);   // T[(q*n3+l)*3+d]
  for (int k = 0; k < n; ++k) for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i)
    for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
      int64_t q = i + n * (j + n * k), l = a + n * (b + n * c);
      grad_phi(L.B, i, j, k, a, b, c, &T[(q * n3 + l) * 3]);
    }
  for (int64_t l = 0; l < n3; ++l)
    for (int64_t m = 0; m < n3; ++m) {
      double s = 0.0;
      for (int64_t q = 0; q < n3; ++q) {
        const double* dl = &T[(q * n3 + l) * 3];
        const double* dm = &T[(q * n3 + m) * 3];
        double g00 = G[0 * n3 + q], g01 = G[1 * n3 + q], g02 = G[2 * n3 + q];
        double g11 = G[3 * n3 + q], g12 = G[4 * n3 + q], g22 = G[5 * n3 + q];
        s += dl[0] * (g00 * dm[0] + g01 * dm[1] + g02 * dm[2])
           + dl[1] * (g01 * dm[0] + g11 * dm[1] + g12 * dm[2])
           + dl[2] * (g02 * dm[0] + g12 * dm[1] + g22 * dm[2]);
      }
      K[l * n3 + m] = s;
    }
}

// Diagonal of the element matrix by the same definition, n^6 per element.
void element_diag(const Level& L, const double* G, double* d) {
  int n = L.n; int64_t n3 = L.n3;
  for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
    int64_t l = a + n * (b + n * c);
    double s = 0.0;
    for (int k = 0; k < n; ++k) for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) {
      int64_t q = i + n * (j + n * k);
      double dl[3];
      grad_phi(L.B, i, j, k, a, b, c, dl);
      double g00 = G[0 * n3 + q], g01 = G[1 * n3 + q], g02 = G[2 * n3 + q];
      double g11 = G[3 * n3 + q], g12 = G[4 * n3 + q], g22 = G[5 * n3 + q];
      s += dl[0] * (g00 * dl[0] + g01 * dl[1] + g02 * dl[2])
         + dl[1] * (g01 * dl[0] + g11 * dl[1] + g12 * dl[2])
         + dl[2] * (g02 * dl[0] + g12 * dl[1] + g22 * dl[2]);
    }
    d[l] = s;
  }
}

/* ------------------------------------------------------------------ global operators */

// A_D u = M A M u + (I - M) u for bc = 0 (R4); A u for bc = 1 (no boundary projection).
void apply(const Level& L, int bc, const double* u, double* v, int tier) {
  int n = L.n; int64_t n3 = L.n3;
  std::vector<double> um(u, u + L.N);
  if (bc == 0)
    for (int64_t g = 0; g < L.N; ++g) if (L.boundary(g)) um[g] = 0.0;
  for (int64_t g = 0; g < L.N; ++g) v[g] = 0.0;
  for (int col = 0; col < 8; ++col) {
    const std::vector<int64_t>& els = L.colour_elems[col];
#pragma omp parallel
    {
      std::vector<double> ue(n3), ve(n3), gbuf;
#pragma omp for schedule(static)
      for (int64_t t = 0; t < (int64_t)els.size(); ++t) {
        int64_t e = els[t];
        for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
          ue[a + n * (b + n * c)] = um[L.l2g(e, a, b, c)];
        const double* G = elem_G(L, e, gbuf);
        if (tier == 2 || L.B.quad == 1) element_apply_o2(L, G, ue.data(), ve.data());
        else element_apply_o3(L, G, ue.data(), ve.data());
        for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
          v[L.l2g(e, a, b, c)] += ve[a + n * (b + n * c)];
      }
    }
  }
  if (bc == 0)
    for (int64_t g = 0; g < L.N; ++g) if (L.boundary(g)) v[g] = u[g];
}

void compute_diag(const Level& L, int bc, double* d) {
  int n = L.n; int64_t n3 = L.n3;
  for (int64_t g = 0; g < L.N; ++g) d[g] = 0.0;
  for (int col = 0; col < 8; ++col) {
    const std::vector<int64_t>& els = L.colour_elems[col];
#pragma omp parallel
    {
      std::vector<double> de(n3), gbuf;
#pragma omp for schedule(static)
      for (int64_t t = 0; t < (int64_t)els.size(); ++t) {
        int64_t e = els[t];
        const double* G = elem_G(L, e, gbuf);
        element_diag(L, G, de.data());
        for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
          d[L.l2g(e, a, b, c)] += de[a + n * (b + n * c)];
      }
    }
  }
  if (bc == 0)
    for (int64_t g = 0; g < L.N; ++g) if (L.boundary(g)) d[g] = 1.0;
}

const std::vector<double>& level_diag(Level& L) {
  if (L.diag_cache.empty()) {
    L.diag_cache.resize(L.N);
    compute_diag(L, 0, L.diag_cache.data());
  }
  return L.diag_cache;
}

double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double nrm2(const std::vector<double>& a) { return std::sqrt(dot(a, a)); }

// R9: power iteration on D^{-1} A_D with the D-Rayleigh quotient; start = splitmix64(seed)
// uniform in [-1,1], boundary zeroed; exactly `iters` applies.
template <class LV>
double lambda_max(LV& L, int iters, uint64_t seed, int64_t* applies) {
  const std::vector<double>& d = level_diag(L);
  std::vector<double> x(L.N), y(L.N);
  for (int64_t g = 0; g < L.N; ++g) x[g] = L.boundary(g) ? 0.0 : uniform_pm1(seed, (uint64_t)g);
  double lam = 0.0;
  for (int it = 0; it < iters; ++it) {
    apply(L, 0, x.data(), y.data(), L.tier);
    if (applies) ++*applies;
    double xy = 0.0, xdx = 0.0;
    for (int64_t g = 0; g < L.N; ++g) { xy += x[g] * y[g]; xdx += x[g] * d[g] * x[g]; }
    lam = xy / xdx;
    for (int64_t g = 0; g < L.N; ++g) y[g] = y[g] / d[g];
    double nz = nrm2(y);
    for (int64_t g = 0; g < L.N; ++g) x[g] = y[g] / nz;
  }
  return lam;
}

// R7: Chebyshev acceleration of Jacobi on D^{-1}A_D over [lo, hi],
// K steps = K applies, written in the residual / correction form.
template <class LV>
void chebyshev(LV& L, const double* b, double* x, int K, double lo, double hi, int64_t* applies) {
  const std::vector<double>& d = level_diag(L);
  int64_t N = L.N;
  double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho = 1.0 / sigma;
  std::vector<double> r(N), Ad(N), dl(N);
  apply(L, 0, x, Ad.data(), L.tier);
  if (applies) ++*applies;
  for (int64_t g = 0; g < N; ++g) { r[g] = b[g] - Ad[g]; dl[g] = r[g] / d[g] / theta; }
  for (int k = 0; k < K; ++k) {
    for (int64_t g = 0; g < N; ++g) x[g] += dl[g];
    if (k == K - 1) break;
    apply(L, 0, dl.data(), Ad.data(), L.tier);
    if (applies) ++*applies;
    double rho_new = 1.0 / (2.0 * sigma - rho);
    for (int64_t g = 0; g < N; ++g) {
      r[g] -= Ad[g];
      dl[g] = rho_new * rho * dl[g] + (2.0 * rho_new / delta) * (r[g] / d[g]);
    }
    rho = rho_new;
  }
}

/* ------------------------------------------------------------------ p-transfer */

// Lowest-index element containing lattice coordinate I along one axis, and the local index.
inline void owner_1d(int64_t I, int p, int& ex, int& a) {
  if (I > 0 && I % p == 0) { ex = (int)(I / p) - 1; a = p; }
  else { ex = (int)(I / p); a = (int)(I - (int64_t)ex * p); }
}

// eq. (7): P_gJ = phi^{coarse}_J(xi(g)) in the canonical (lowest-index) element of g;
// P0 = M_f P M_c (R12).  Direct definition, one fine node at a time.
void prolong(const Level& C, const Level& F, const double* uc, double* uf) {
  int nc = C.n, nf = F.n;
  std::vector<double> I(nf * nc);
  for (int i = 0; i < nf; ++i)
    for (int a = 0; a < nc; ++a) I[i * nc + a] = lagrange(C.B.x, a, F.B.x[i]);
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) { uf[g] = 0.0; continue; }
    int64_t IX = g % F.Mx, JY = (g / F.Mx) % F.My, KZ = g / (F.Mx * F.My);
    int ex, ey, ez, i, j, k;
    owner_1d(IX, F.p, ex, i); owner_1d(JY, F.p, ey, j); owner_1d(KZ, F.p, ez, k);
    int64_t e = ex + (int64_t)C.nex * (ey + (int64_t)C.ney * ez);
    double s = 0.0;
    for (int c = 0; c < nc; ++c) for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      int64_t gc = C.l2g(e, a, b, c);
      double ucm = C.boundary(gc) ? 0.0 : uc[gc];
      s += I[i * nc + a] * I[j * nc + b] * I[k * nc + c] * ucm;
    }
    uf[g] = s;
  }
}

// R = P0^T: every fine node contributes once, through its canonical element (R12).
void restrict_(const Level& C, const Level& F, const double* rf, double* rc) {
  int nc = C.n, nf = F.n;
  std::vector<double> I(nf * nc);
  for (int i = 0; i < nf; ++i)
    for (int a = 0; a < nc; ++a) I[i * nc + a] = lagrange(C.B.x, a, F.B.x[i]);
  for (int64_t g = 0; g < C.N; ++g) rc[g] = 0.0;
  for (int col = 0; col < 8; ++col) {
    const std::vector<int64_t>& els = F.colour_elems[col];
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)els.size(); ++t) {
      int64_t e = els[t];
      int ex, ey, ez; F.elem_coords(e, ex, ey, ez);
      for (int k = 0; k < nf; ++k) for (int j = 0; j < nf; ++j) for (int i = 0; i < nf; ++i) {
        if ((i == 0 && ex > 0) || (j == 0 && ey > 0) || (k == 0 && ez > 0)) continue; // not owner
        int64_t g = F.l2g(e, i, j, k);
        if (F.boundary(g)) continue;
        double val = rf[g];
        for (int c = 0; c < nc; ++c) for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a)
          rc[C.l2g(e, a, b, c)] += I[i * nc + a] * I[j * nc + b] * I[k * nc + c] * val;
      }
    }
  }
  for (int64_t g = 0; g < C.N; ++g) if (C.boundary(g)) rc[g] = 0.0;
}

/* ------------------------------------------------------------------ h-transfer */

// Position of fine lattice coordinate I (one axis) in the coarse element grid: the reference-cube
// coordinate X = (e_f + (xhat^F_i + 1)/2) / ne_f of the fine node, the canonical (lowest-index)
// coarse element e_c containing it and the local coordinate xi in [-1, 1] (R25: the element grids
// are nested in reference-lattice coordinates).
inline void h_position(int64_t I, int pf, const std::vector<double>& xf, int nef, int nec, int& ec, double& xi) {
  int ef, i;
  owner_1d(I, pf, ef, i);
  const double X = (ef + 0.5 * (xf[i] + 1.0)) / nef;
  const double t = X * nec;
  double fl = std::floor(t);
  ec = (int)fl;
  if (t == fl && ec > 0) ec -= 1;   // on a coarse element face: the lower element
  if (ec >= nec) ec = nec - 1;
  xi = 2.0 * (t - ec) - 1.0;
}

// eq. (7) across meshes: P_gJ = phi^C_J(X(g)), C and F of the same order with F.ne = 2 C.ne; P0 =
// M_f P M_c (R12).  Direct definition, one fine node at a time.
void prolong_h(const Level& C, const Level& F, const double* uc, double* uf) {
  const int nc = C.n;
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) { uf[g] = 0.0; continue; }
    int64_t IX = g % F.Mx, JY = (g / F.Mx) % F.My, KZ = g / (F.Mx * F.My);
    int ex, ey, ez;
    double xi, eta, zeta;
    h_position(IX, F.p, F.B.x, F.nex, C.nex, ex, xi);
    h_position(JY, F.p, F.B.x, F.ney, C.ney, ey, eta);
    h_position(KZ, F.p, F.B.x, F.nez, C.nez, ez, zeta);
    int64_t e = ex + (int64_t)C.nex * (ey + (int64_t)C.ney * ez);
    double s = 0.0;
    for (int c = 0; c < nc; ++c) for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      int64_t gc = C.l2g(e, a, b, c);
      if (C.boundary(gc)) continue;
      s += lagrange(C.B.x, a, xi) * lagrange(C.B.x, b, eta) * lagrange(C.B.x, c, zeta) * uc[gc];
    }
    uf[g] = s;
  }
}

// R = P0^T for the h pair: every interior fine node adds P_gJ r_g to the interior coarse nodes J
// of its canonical coarse element (sequential: the h-levels are small).
void restrict_h(const Level& C, const Level& F, const double* rf, double* rc) {
  const int nc = C.n;
  for (int64_t g = 0; g < C.N; ++g) rc[g] = 0.0;
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) continue;
    int64_t IX = g % F.Mx, JY = (g / F.Mx) % F.My, KZ = g / (F.Mx * F.My);
    int ex, ey, ez;
    double xi, eta, zeta;
    h_position(IX, F.p, F.B.x, F.nex, C.nex, ex, xi);
    h_position(JY, F.p, F.B.x, F.ney, C.ney, ey, eta);
    h_position(KZ, F.p, F.B.x, F.nez, C.nez, ez, zeta);
    int64_t e = ex + (int64_t)C.nex * (ey + (int64_t)C.ney * ez);
    for (int c = 0; c < nc; ++c) for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      int64_t gc = C.l2g(e, a, b, c);
      if (C.boundary(gc)) continue;
      rc[gc] += lagrange(C.B.x, a, xi) * lagrange(C.B.x, b, eta) * lagrange(C.B.x, c, zeta) * rf[g];
    }
  }
}

// Level pair kind: 1 = p pair (F.p = 2 C.p, same mesh), 2 = h pair (same p, F.ne = 2 C.ne), 0 = neither.
int pair_kind(const Level& C, const Level& F) {
  const bool same_mesh = C.nex == F.nex && C.ney == F.ney && C.nez == F.nez;
  if (same_mesh && F.p == 2 * C.p) return 1;
  if (C.p == F.p && F.nex == 2 * C.nex && F.ney == 2 * C.ney && F.nez == 2 * C.nez) return 2;
  return 0;
}
void transfer_prolong(const Level& C, const Level& F, const double* uc, double* uf) {
  if (pair_kind(C, F) == 2) prolong_h(C, F, uc, uf); else prolong(C, F, uc, uf);
}
void transfer_restrict(const Level& C, const Level& F, const double* rf, double* rc) {
  if (pair_kind(C, F) == 2) restrict_h(C, F, rf, rc); else restrict_(C, F, rf, rc);
}

/* ------------------------------------------------------------------ NEXT-1 smoother / estimator */

// Damped point Jacobi, omega = 2/3 in the paper:
// x <- x + omega D^{-1} (b - A_D x); one apply per step.
template <class LV>
void jacobi(LV& L, const double* b, double* x, int steps, double omega, int64_t* applies) {
  const std::vector<double>& d = level_diag(L);
  std::vector<double> Ax(L.N);
  for (int s = 0; s < steps; ++s) {
    apply(L, 0, x, Ax.data(), L.tier);
    if (applies) ++*applies;
    for (int64_t g = 0; g < L.N; ++g) x[g] += omega * (b[g] - Ax[g]) / d[g];
  }
}

// Eigenvalues of a small symmetric matrix (row-major, n x n) by cyclic Jacobi rotations.
void sym_eig_jacobi(int n, std::vector<double> A, std::vector<double>& ev) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) if (i != j) off += A[i * n + j] * A[i * n + j];
    if (off < 1e-30) break;
    for (int pp = 0; pp < n - 1; ++pp)
      for (int q = pp + 1; q < n; ++q) {
        double apq = A[pp * n + q];
        if (apq == 0.0) continue;
        double theta = (A[q * n + q] - A[pp * n + pp]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < n; ++k) {   // A <- J^T A J
          double akp = A[k * n + pp], akq = A[k * n + q];
          A[k * n + pp] = c * akp - sn * akq;
          A[k * n + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = A[pp * n + k], aqk = A[q * n + k];
          A[pp * n + k] = c * apk - sn * aqk;
          A[q * n + k] = sn * apk + c * aqk;
        }
      }
  }
  ev.resize(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
}

// lambda_max(D^{-1} A_D) from m Arnoldi iterations (reading R26): Arnoldi with
// modified Gram-Schmidt in the D-inner product <x, y>_D = sum d x y, in which D^{-1}A_D is
// self-adjoint; start = splitmix64(seed) uniform in [-1,1] with the boundary zeroed (R9).  The
// estimate is the largest eigenvalue of the k x k Hessenberg matrix H (k = m, or fewer on an
// invariant subspace), symmetric tridiagonal up to rounding; its symmetric part is diagonalised.
template <class LV>
double lambda_arnoldi(LV& L, int m, uint64_t seed, int64_t* applies) {
  const std::vector<double>& d = level_diag(L);
  const int64_t N = L.N;
  auto dotD = [&](const std::vector<double>& a, const std::vector<double>& b) {
    double s = 0.0;
    for (int64_t g = 0; g < N; ++g) s += d[g] * a[g] * b[g];
    return s;
  };
  std::vector<std::vector<double>> V;
  std::vector<double> v(N), w(N), Aw(N);
  for (int64_t g = 0; g < N; ++g) v[g] = L.boundary(g) ? 0.0 : uniform_pm1(seed, (uint64_t)g);
  double nv = std::sqrt(dotD(v, v));
  for (int64_t g = 0; g < N; ++g) v[g] /= nv;
  V.push_back(v);
  std::vector<double> H((m + 1) * m, 0.0);   // H[i*m + j]
  int k = 0;
  for (int j = 0; j < m; ++j) {
    apply(L, 0, V[j].data(), Aw.data(), L.tier);
    if (applies) ++*applies;
    for (int64_t g = 0; g < N; ++g) w[g] = Aw[g] / d[g];
    const double wn0 = std::sqrt(dotD(w, w));
    for (int pass = 0; pass < 2; ++pass)   // modified Gram-Schmidt, repeated once ("twice is enough")
      for (int i = 0; i <= j; ++i) {
        double h = dotD(w, V[i]);
        H[i * m + j] += h;
        for (int64_t g = 0; g < N; ++g) w[g] -= h * V[i][g];
      }
    k = j + 1;
    double hn = std::sqrt(dotD(w, w));
    H[(j + 1) * m + j] = hn;
    if (hn <= 1e-10 * wn0) break;   // invariant subspace reached (Krylov space exhausted)
    for (int64_t g = 0; g < N; ++g) w[g] /= hn;
    V.push_back(w);
  }
  std::vector<double> S(k * k), ev;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) S[i * k + j] = 0.5 * (H[i * m + j] + H[j * m + i]);
  sym_eig_jacobi(k, S, ev);
  double lam = ev[0];
  for (double e : ev) lam = std::max(lam, e);
  return lam;
}

/* ------------------------------------------------------------------ hierarchy / solvers */

template <class LV>
struct HierT {
  std::vector<LV*> lv;      // lv[0] finest (order p), lv.back() the coarsest level
  std::vector<double> lam;
  int nu_pre, nu_post, K;
  double lo_frac, hi_frac, coarse_rtol;
  int coarse_maxit, power_iters;
  uint64_t seed;
  int smoother = 0;          // 0 Chebyshev-Jacobi (degree K), 1 damped point Jacobi (omega)
  double omega = 2.0 / 3.0;
  int lambda_method = 0;     // 0 power iteration (R9), 1 Arnoldi (R26)
  int64_t fine_applies = 0;
  int64_t coarse_iters_last = 0;
};
using Hier = HierT<Level>;

template <class H_>
int64_t* counter_for(H_& H, int l) { return l == 0 ? &H.fine_applies : nullptr; }

// R13: unpreconditioned CG on the coarsest level, x0 = 0, ||r|| <= rtol ||b||.
template <class LV>
int coarse_cg(HierT<LV>& H, const double* b, double* x) {
  LV& L = *H.lv.back();
  int64_t N = L.N;
  int l = (int)H.lv.size() - 1;
  std::vector<double> r(b, b + N), p(b, b + N), Ap(N);
  for (int64_t g = 0; g < N; ++g) x[g] = 0.0;
  double bn = nrm2(r);
  H.coarse_iters_last = 0;
  if (bn == 0.0) return 0;
  double rr = dot(r, r);
  for (int it = 0; it < H.coarse_maxit; ++it) {
    if (std::sqrt(rr) <= H.coarse_rtol * bn) break;
    apply(L, 0, p.data(), Ap.data(), L.tier);
    if (int64_t* c = counter_for(H, l)) ++*c;
    double pAp = dot(p, Ap);
    if (pAp <= 0.0) return 6;
    double alpha = rr / pAp;
    for (int64_t g = 0; g < N; ++g) { x[g] += alpha * p[g]; r[g] -= alpha * Ap[g]; }
    double rr_new = dot(r, r);
    double beta = rr_new / rr;
    for (int64_t g = 0; g < N; ++g) p[g] = r[g] + beta * p[g];
    rr = rr_new;
    ++H.coarse_iters_last;
  }
  return 0;
}

// V-cycle from x = 0 (R11).
template <class LV>
int vcycle(HierT<LV>& H, int l, const double* b, double* x) {
  LV& L = *H.lv[l];
  int64_t N = L.N;
  if (l == (int)H.lv.size() - 1) return coarse_cg(H, b, x);
  for (int64_t g = 0; g < N; ++g) x[g] = 0.0;
  double lo = H.lo_frac * H.lam[l], hi = H.hi_frac * H.lam[l];
  // one smoothing application: a degree-K Chebyshev polynomial, or one damped Jacobi step
  auto smooth = [&]() {
    if (H.smoother == 1) jacobi(L, b, x, 1, H.omega, counter_for(H, l));
    else chebyshev(L, b, x, H.K, lo, hi, counter_for(H, l));
  };
  for (int s = 0; s < H.nu_pre; ++s) smooth();
  std::vector<double> r(N);
  apply(L, 0, x, r.data(), L.tier);
  if (int64_t* c = counter_for(H, l)) ++*c;
  for (int64_t g = 0; g < N; ++g) r[g] = b[g] - r[g];
  LV& C = *H.lv[l + 1];
  std::vector<double> bc(C.N), ec(C.N), ef(N);
  transfer_restrict(C, L, r.data(), bc.data());
  int st = vcycle(H, l + 1, bc.data(), ec.data());
  if (st) return st;
  transfer_prolong(C, L, ec.data(), ef.data());
  for (int64_t g = 0; g < N; ++g) x[g] += ef[g];
  for (int s = 0; s < H.nu_post; ++s) smooth();
  return 0;
}

/* ================================================================== NEXT-2: 2-D quadrilaterals */
// The 2-D problems of the paper: -div(mu grad u) = f on the unit square (2d-const) or a
// warped square (2d-var, 2d-var'), with the same discretisation as in 3-D: tensor LGL
// nodal basis of order p on quadrilaterals, isoparametric geometry, Gauss or collocated LGL
// quadrature (R1 / NEXT-3).  Written separately from the 3-D level (no shared element code); the
// smoothers, eigenvalue estimates, hierarchy and solvers above are templates over the level type.

// mu in 2-D (R6): 0: c0 (2d-const); 1: exp(c1 S), 2: 10^(c1 S), S = sin 2 pi x sin 2 pi y;
// 3: c0 + c1 (cos^2 2 pi x + cos^2 2 pi y) (2d-var, c0 = 1, c1 = 1e6); 4: c0 + c1 (cos^2 10 pi x +
// cos^2 10 pi y) (2d-var').
double coeff_mu2(int kind, double c0, double c1, double x, double y) {
  const double S = std::sin(2 * kPi * x) * std::sin(2 * kPi * y);
  switch (kind) {
    case 0: return c0;
    case 1: return std::exp(c1 * S);
    case 2: return std::pow(10.0, c1 * S);
    case 3: { double a = std::cos(2 * kPi * x), b = std::cos(2 * kPi * y); return c0 + c1 * (a * a + b * b); }
    case 4: { double a = std::cos(10 * kPi * x), b = std::cos(10 * kPi * y); return c0 + c1 * (a * a + b * b); }
  }
  return NAN;
}
void coeff_grad2(int kind, double c0, double c1, double x, double y, double g[2]) {
  const double dS[2] = {2 * kPi * std::cos(2 * kPi * x) * std::sin(2 * kPi * y),
                        2 * kPi * std::sin(2 * kPi * x) * std::cos(2 * kPi * y)};
  const double mu = coeff_mu2(kind, c0, c1, x, y);
  switch (kind) {
    case 0: g[0] = g[1] = 0.0; return;
    case 1: g[0] = c1 * mu * dS[0]; g[1] = c1 * mu * dS[1]; return;
    case 2: g[0] = std::log(10.0) * c1 * mu * dS[0]; g[1] = std::log(10.0) * c1 * mu * dS[1]; return;
    case 3: g[0] = -2 * kPi * c1 * std::sin(4 * kPi * x); g[1] = -2 * kPi * c1 * std::sin(4 * kPi * y); return;
    case 4: g[0] = -10 * kPi * c1 * std::sin(20 * kPi * x); g[1] = -10 * kPi * c1 * std::sin(20 * kPi * y); return;
  }
}

struct Level2 {
  int nex, ney, p, n, warp, coeff;
  double amp, c0, c1;
  int64_t E, N, Mx, My, n2;
  int tier = 2;                    // (one apply tier in 2-D: direct quadrature)
  Basis B;
  std::vector<double> G;           // [E][3][n2] at the quadrature points: (00, 01, 11)
  std::vector<double> detJ;        // [E][n2]
  std::vector<double> diag_cache;
  std::vector<std::vector<int64_t>> colour_elems;   // 4 colours, (ex & 1) | (ey & 1) << 1
  double min_detj = 1e300;
  int status = 0;
  void elem_coords(int64_t e, int& ex, int& ey) const { ex = (int)(e % nex); ey = (int)(e / nex); }
  int64_t l2g(int64_t e, int a, int b) const {
    int ex, ey; elem_coords(e, ex, ey);
    return ((int64_t)ex * p + a) + Mx * ((int64_t)ey * p + b);
  }
  bool boundary(int64_t g) const {
    int64_t I = g % Mx, J = g / Mx;
    return I == 0 || I == Mx - 1 || J == 0 || J == My - 1;
  }
};

// Physical node coordinates of element e: reference-square point, then x_i += a sin(pi X) sin(pi Y)
// (the 2-D analogue of the BASELINE warp; the paper's own warped square is unpublished, R5).
void element_nodes2(const Level2& L, int64_t e, std::vector<double>& X) {
  const int n = L.n;
  X.assign(2 * L.n2, 0.0);
  int ex, ey; L.elem_coords(e, ex, ey);
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < n; ++a) {
      const int l = a + n * b;
      const double Xr = (ex + 0.5 * (L.B.x[a] + 1.0)) / L.nex, Yr = (ey + 0.5 * (L.B.x[b] + 1.0)) / L.ney;
      const double s = (L.warp == 1) ? L.amp * std::sin(kPi * Xr) * std::sin(kPi * Yr) : 0.0;
      X[l] = Xr + s; X[L.n2 + l] = Yr + s;
    }
}

// grad_ref phi_(a,b) at quadrature point (i,j) from the 1-D tabulations.
inline void grad_phi2(const Basis& B, int i, int j, int a, int b, double d[2]) {
  const int n = B.n;
  d[0] = B.dL[i * n + a] * B.L[j * n + b];
  d[1] = B.L[i * n + a] * B.dL[j * n + b];
}

// G_q = w_i w_j mu(x_q) detJ_q J_q^{-1} J_q^{-T}, J = d x / d xi by the definition
// J[al][be] = sum_l x_l^al d_be phi_l(xi_q).  Returns min det J.
double element_geometry2(const Level2& L, int64_t e, double* G, double* dJ) {
  const int n = L.n; const int64_t n2 = L.n2;
  std::vector<double> X;
  element_nodes2(L, e, X);
  double mind = 1e300;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int q = i + n * j;
      double J[2][2] = {{0, 0}, {0, 0}}, xq[2] = {0, 0};
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          const int l = a + n * b;
          double d[2];
          grad_phi2(L.B, i, j, a, b, d);
          for (int al = 0; al < 2; ++al)
            for (int be = 0; be < 2; ++be) J[al][be] += X[al * n2 + l] * d[be];
          const double ph = L.B.L[i * n + a] * L.B.L[j * n + b];
          xq[0] += ph * X[l]; xq[1] += ph * X[n2 + l];
        }
      const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      mind = std::min(mind, det);
      const double Ji[2][2] = {{J[1][1] / det, -J[0][1] / det}, {-J[1][0] / det, J[0][0] / det}};
      const double s = L.B.qw[i] * L.B.qw[j] * coeff_mu2(L.coeff, L.c0, L.c1, xq[0], xq[1]) * det;
      G[0 * n2 + q] = s * (Ji[0][0] * Ji[0][0] + Ji[0][1] * Ji[0][1]);
      G[1 * n2 + q] = s * (Ji[0][0] * Ji[1][0] + Ji[0][1] * Ji[1][1]);
      G[2 * n2 + q] = s * (Ji[1][0] * Ji[1][0] + Ji[1][1] * Ji[1][1]);
      if (dJ) dJ[q] = det;
    }
  return mind;
}

// Direct quadrature (O2): v_l = sum_q grad phi_l(q)^T G_q sum_m u_m grad phi_m(q).
void element_apply2(const Level2& L, const double* G, const double* u, double* v) {
  const int n = L.n; const int64_t n2 = L.n2;
  for (int64_t l = 0; l < n2; ++l) v[l] = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int q = i + n * j;
      double g[2] = {0, 0};
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          double d[2];
          grad_phi2(L.B, i, j, a, b, d);
          g[0] += d[0] * u[a + n * b]; g[1] += d[1] * u[a + n * b];
        }
      const double w0 = G[q] * g[0] + G[n2 + q] * g[1], w1 = G[n2 + q] * g[0] + G[2 * n2 + q] * g[1];
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          double d[2];
          grad_phi2(L.B, i, j, a, b, d);
          v[a + n * b] += d[0] * w0 + d[1] * w1;
        }
    }
}

// Dense element matrix K[l][m] = sum_q grad phi_l(q)^T G_q grad phi_m(q).
void element_matrix2(const Level2& L, const double* G, double* K) {
  const int n = L.n; const int64_t n2 = L.n2;
  for (int64_t l = 0; l < n2; ++l)
    for (int64_t m = 0; m < n2; ++m) {
      double s = 0.0;
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const int q = i + n * j;
          double dl[2], dm[2];
          grad_phi2(L.B, i, j, (int)(l % n), (int)(l / n), dl);
          grad_phi2(L.B, i, j, (int)(m % n), (int)(m / n), dm);
          s += dl[0] * (G[q] * dm[0] + G[n2 + q] * dm[1]) + dl[1] * (G[n2 + q] * dm[0] + G[2 * n2 + q] * dm[1]);
        }
      K[l * n2 + m] = s;
    }
}

void element_diag2(const Level2& L, const double* G, double* d) {
  const int n = L.n; const int64_t n2 = L.n2;
  for (int64_t l = 0; l < n2; ++l) {
    double s = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int q = i + n * j;
        double dl[2];
        grad_phi2(L.B, i, j, (int)(l % n), (int)(l / n), dl);
        s += dl[0] * (G[q] * dl[0] + G[n2 + q] * dl[1]) + dl[1] * (G[n2 + q] * dl[0] + G[2 * n2 + q] * dl[1]);
      }
    d[l] = s;
  }
}

// A_D u = M A M u + (I - M) u (bc 0, R4); A u (bc 1).
void apply(const Level2& L, int bc, const double* u, double* v, int) {
  const int n = L.n; const int64_t n2 = L.n2;
  std::vector<double> um(u, u + L.N);
  if (bc == 0)
    for (int64_t g = 0; g < L.N; ++g) if (L.boundary(g)) um[g] = 0.0;
  for (int64_t g = 0; g < L.N; ++g) v[g] = 0.0;
  for (int col = 0; col < 4; ++col) {
    const std::vector<int64_t>& els = L.colour_elems[col];
#pragma omp parallel
    {
      std::vector<double> ue(n2), ve(n2);
#pragma omp for schedule(static)
      for (int64_t t = 0; t < (int64_t)els.size(); ++t) {
        const int64_t e = els[t];
        for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) ue[a + n * b] = um[L.l2g(e, a, b)];
        element_apply2(L, &L.G[(size_t)e * 3 * n2], ue.data(), ve.data());
        for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) v[L.l2g(e, a, b)] += ve[a + n * b];
      }
    }
  }
  if (bc == 0)
    for (int64_t g = 0; g < L.N; ++g) if (L.boundary(g)) v[g] = u[g];
}

void compute_diag(const Level2& L, int bc, double* d) {
  const int n = L.n; const int64_t n2 = L.n2;
  for (int64_t g = 0; g < L.N; ++g) d[g] = 0.0;
  std::vector<double> de(n2);
  for (int64_t e = 0; e < L.E; ++e) {
    element_diag2(L, &L.G[(size_t)e * 3 * n2], de.data());
    for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) d[L.l2g(e, a, b)] += de[a + n * b];
  }
  if (bc == 0)
    for (int64_t g = 0; g < L.N; ++g) if (L.boundary(g)) d[g] = 1.0;
}

const std::vector<double>& level_diag(Level2& L) {
  if (L.diag_cache.empty()) {
    L.diag_cache.resize(L.N);
    compute_diag(L, 0, L.diag_cache.data());
  }
  return L.diag_cache;
}

// p-transfer (eq. (7)): P_gJ = phi^C_J(xi(g)) in the canonical element of fine node g; P0 = M_f P M_c.
void prolong(const Level2& C, const Level2& F, const double* uc, double* uf) {
  const int nc = C.n;
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) { uf[g] = 0.0; continue; }
    int ex, ey, i, j;
    owner_1d(g % F.Mx, F.p, ex, i); owner_1d(g / F.Mx, F.p, ey, j);
    const int64_t e = ex + (int64_t)C.nex * ey;
    double s = 0.0;
    for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      const int64_t gc = C.l2g(e, a, b);
      if (!C.boundary(gc)) s += lagrange(C.B.x, a, F.B.x[i]) * lagrange(C.B.x, b, F.B.x[j]) * uc[gc];
    }
    uf[g] = s;
  }
}
// R = P0^T: each interior fine node adds P_gJ r_g to the interior coarse nodes of its canonical element.
void restrict_(const Level2& C, const Level2& F, const double* rf, double* rc) {
  const int nc = C.n;
  for (int64_t g = 0; g < C.N; ++g) rc[g] = 0.0;
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) continue;
    int ex, ey, i, j;
    owner_1d(g % F.Mx, F.p, ex, i); owner_1d(g / F.Mx, F.p, ey, j);
    const int64_t e = ex + (int64_t)C.nex * ey;
    for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      const int64_t gc = C.l2g(e, a, b);
      if (!C.boundary(gc)) rc[gc] += lagrange(C.B.x, a, F.B.x[i]) * lagrange(C.B.x, b, F.B.x[j]) * rf[g];
    }
  }
}
// h-transfer (eq. (7) across nested meshes, R25): the coarse basis at the fine node's reference position.
void prolong_h(const Level2& C, const Level2& F, const double* uc, double* uf) {
  const int nc = C.n;
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) { uf[g] = 0.0; continue; }
    int ex, ey; double xi, eta;
    h_position(g % F.Mx, F.p, F.B.x, F.nex, C.nex, ex, xi);
    h_position(g / F.Mx, F.p, F.B.x, F.ney, C.ney, ey, eta);
    const int64_t e = ex + (int64_t)C.nex * ey;
    double s = 0.0;
    for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      const int64_t gc = C.l2g(e, a, b);
      if (!C.boundary(gc)) s += lagrange(C.B.x, a, xi) * lagrange(C.B.x, b, eta) * uc[gc];
    }
    uf[g] = s;
  }
}
void restrict_h(const Level2& C, const Level2& F, const double* rf, double* rc) {
  const int nc = C.n;
  for (int64_t g = 0; g < C.N; ++g) rc[g] = 0.0;
  for (int64_t g = 0; g < F.N; ++g) {
    if (F.boundary(g)) continue;
    int ex, ey; double xi, eta;
    h_position(g % F.Mx, F.p, F.B.x, F.nex, C.nex, ex, xi);
    h_position(g / F.Mx, F.p, F.B.x, F.ney, C.ney, ey, eta);
    const int64_t e = ex + (int64_t)C.nex * ey;
    for (int b = 0; b < nc; ++b) for (int a = 0; a < nc; ++a) {
      const int64_t gc = C.l2g(e, a, b);
      if (!C.boundary(gc)) rc[gc] += lagrange(C.B.x, a, xi) * lagrange(C.B.x, b, eta) * rf[g];
    }
  }
}
int pair_kind(const Level2& C, const Level2& F) {
  if (C.nex == F.nex && C.ney == F.ney && F.p == 2 * C.p) return 1;
  if (C.p == F.p && F.nex == 2 * C.nex && F.ney == 2 * C.ney) return 2;
  return 0;
}
void transfer_prolong(const Level2& C, const Level2& F, const double* uc, double* uf) {
  if (pair_kind(C, F) == 2) prolong_h(C, F, uc, uf); else prolong(C, F, uc, uf);
}
void transfer_restrict(const Level2& C, const Level2& F, const double* rf, double* rc) {
  if (pair_kind(C, F) == 2) restrict_h(C, F, rf, rc); else restrict_(C, F, rf, rc);
}

using Hier2 = HierT<Level2>;

// mode 0: MG as solver x <- x + V(b - A x); mode 1: MG-preconditioned CG (Algorithm 1,
// P:973-991).  x0 = 0 (R14); stop at ||r||_2 <= rtol ||r0||_2.
// Divergence (||r|| > 10 ||r0||) stops with converged = 0.
template <class LV>
int solve_impl(HierT<LV>* H, int mode, const double* b, double* x, double rtol, int maxit,
               int* iters_out, int* converged, double* r0n, double* rn, double* hist, int hist_cap,
               int64_t* fine_applies) {
  LV& L = *H->lv[0];
  int64_t N = L.N;
  H->fine_applies = 0;
  std::vector<double> r(b, b + N), z(N), pv(N), hv(N);
  for (int64_t g = 0; g < N; ++g) x[g] = 0.0;
  double r0 = nrm2(r), rnorm = r0;
  int it = 0, st = 0;
  *converged = 0;
  if (hist && hist_cap > 0) hist[0] = r0;
  if (r0 == 0.0) { *converged = 1; goto done; }
  if (mode == 0) {
    while (it < maxit) {
      if (rnorm <= rtol * r0) { *converged = 1; break; }
      if (rnorm > 10.0 * r0) break;
      st = vcycle(*H, 0, r.data(), z.data());
      if (st) break;
      for (int64_t g = 0; g < N; ++g) x[g] += z[g];
      apply(L, 0, x, hv.data(), L.tier);
      ++H->fine_applies;
      for (int64_t g = 0; g < N; ++g) r[g] = b[g] - hv[g];
      rnorm = nrm2(r);
      ++it;
      if (hist && it < hist_cap) hist[it] = rnorm;
    }
    if (rnorm <= rtol * r0) *converged = 1;
  } else {
    st = vcycle(*H, 0, r.data(), z.data());
    if (st) goto done;
    pv = z;
    double rho_r = dot(z, r);
    while (it < maxit) {
      apply(L, 0, pv.data(), hv.data(), L.tier);                 // h = A p
      ++H->fine_applies;
      double ph = dot(pv, hv);
      if (ph <= 0.0) { st = 6; break; }
      double alpha = rho_r / ph;
      for (int64_t g = 0; g < N; ++g) { x[g] += alpha * pv[g]; r[g] -= alpha * hv[g]; }
      rnorm = nrm2(r);
      ++it;
      if (hist && it < hist_cap) hist[it] = rnorm;
      if (rnorm <= rtol * r0) { *converged = 1; break; }      // convergence test
      if (rnorm > 10.0 * r0) break;
      st = vcycle(*H, 0, r.data(), z.data());                  // rho = M r
      if (st) break;
      double rho_new = dot(z, r);
      double beta = rho_new / rho_r;
      for (int64_t g = 0; g < N; ++g) pv[g] = z[g] + beta * pv[g];
      rho_r = rho_new;
    }
  }
done:
  *iters_out = it;
  *r0n = r0; *rn = rnorm;
  *fine_applies = H->fine_applies;
  return st;
}

}  // namespace

/* ================================================================== C ABI (ctypes) */
extern "C" {

void orc_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }
// Quadrature of levels created afterwards: 0 collocated LGL (R1, default), 1 Gauss-Legendre with
// p + 1 points per direction (NEXT-3).  Oracle-only: the GPU path is collocated.
void orc_set_quadrature(int q) { g_quad = (q == 1) ? 1 : 0; }
int orc_get_threads(void) { return omp_get_max_threads(); }

int orc_lgl(int p, double* x, double* w) {
  if (p < 1 || p > 64) return 2;
  std::vector<double> xs, ws;
  lgl(p, xs, ws);
  for (int i = 0; i <= p; ++i) { x[i] = xs[i]; if (w) w[i] = ws[i]; }
  return 0;
}

// D[i*n+m] = ell_m'(xhat_i) on the order-p LGL nodes.
int orc_deriv_matrix(int p, double* D) {
  if (p < 1 || p > 64) return 2;
  Basis B; B.build(p);
  std::memcpy(D, B.dL.data(), sizeof(double) * B.n * B.n);
  return 0;
}

// Evaluate all order-p Lagrange cardinals (and derivatives) at t.
int orc_lagrange_eval(int p, double t, double* l, double* dl) {
  if (p < 1 || p > 64) return 2;
  std::vector<double> xs, ws;
  lgl(p, xs, ws);
  for (int m = 0; m <= p; ++m) { l[m] = lagrange(xs, m, t); if (dl) dl[m] = dlagrange(xs, m, t); }
  return 0;
}

// I[i*(pc+1)+a] = ell^{pc}_a(xhat^{pf}_i)  (eq. 7).
int orc_interp_matrix(int pc, int pf, double* I) {
  if (pc < 1 || pf < 1) return 2;
  std::vector<double> xc, wc, xf, wf;
  lgl(pc, xc, wc); lgl(pf, xf, wf);
  for (int i = 0; i <= pf; ++i)
    for (int a = 0; a <= pc; ++a) I[i * (pc + 1) + a] = lagrange(xc, a, xf[i]);
  return 0;
}

uint64_t orc_splitmix64(uint64_t seed, uint64_t i) { return splitmix64_at(seed, i); }

double orc_coeff(int kind, double c0, double c1, double x, double y, double z) {
  return coeff_mu(kind, c0, c1, x, y, z);
}

// Create a level. eager=1 precomputes G for every element (needed for O1/diag caches at
// small sizes); eager=0 recomputes geometry per element on use (large meshes, sampled rows).
void* orc_level_create(int nex, int ney, int nez, int p, int warp, double amp, int coeff,
                       double c0, double c1, int eager, int geom_tier, int tier) {
  if (p < 1 || p > 16 || nex < 1 || ney < 1 || nez < 1) return nullptr;
  Level* L = new Level();
  L->nex = nex; L->ney = ney; L->nez = nez; L->p = p; L->n = p + 1;
  L->warp = warp; L->amp = amp; L->coeff = coeff; L->c0 = c0; L->c1 = c1;
  L->E = (int64_t)nex * ney * nez;
  L->Mx = (int64_t)nex * p + 1; L->My = (int64_t)ney * p + 1; L->Mz = (int64_t)nez * p + 1;
  L->N = L->Mx * L->My * L->Mz;
  L->n3 = (int64_t)L->n * L->n * L->n;
  L->geom_tier = geom_tier; L->tier = tier; L->eager = eager != 0;
  L->B.build(p, g_quad);
  if (g_quad == 1) { L->geom_tier = 2; L->tier = 2; }   // O3 / factorised J assume collocation
  L->colour_elems.assign(8, {});
  for (int64_t e = 0; e < L->E; ++e) {
    int ex, ey, ez; L->elem_coords(e, ex, ey, ez);
    L->colour_elems[(ex & 1) | ((ey & 1) << 1) | ((ez & 1) << 2)].push_back(e);
  }
  if (L->eager) {
    L->G.resize((size_t)L->E * 6 * L->n3);
    L->detJ.resize((size_t)L->E * L->n3);
    double mind = 1e300;
#pragma omp parallel for schedule(dynamic) reduction(min : mind)
    for (int64_t e = 0; e < L->E; ++e) {
      double m = element_geometry(*L, e, &L->G[(size_t)e * 6 * L->n3], &L->detJ[(size_t)e * L->n3],
                                  L->geom_tier);
      mind = std::min(mind, m);
    }
    L->min_detj = mind;
    if (!(mind > 0.0)) L->status = 4;
  }
  return L;
}

void orc_level_destroy(void* h) { delete (Level*)h; }
int orc_level_status(void* h) { return ((Level*)h)->status; }
double orc_level_min_detj(void* h) {
  Level* L = (Level*)h;
  if (!L->eager) {
    double mind = 1e300;
#pragma omp parallel
    {
      std::vector<double> G(6 * L->n3);
#pragma omp for schedule(dynamic) reduction(min : mind)
      for (int64_t e = 0; e < L->E; ++e) mind = std::min(mind, element_geometry(*L, e, G.data(), nullptr, L->geom_tier));
    }
    L->min_detj = mind;
  }
  return L->min_detj;
}
int64_t orc_level_ndofs(void* h) { return ((Level*)h)->N; }
int64_t orc_level_nelem(void* h) { return ((Level*)h)->E; }
void orc_level_set_tier(void* h, int tier) { ((Level*)h)->tier = tier; }

// Lattice-independent numbering by coordinate matching: collect every
// (element, local node) with its reference-cube lattice coordinate, sort, number unique
// coordinates in (z, y, x) lexicographic order.  Pins the closed form used elsewhere.
int orc_l2g_by_matching(void* h, int32_t* l2g) {
  Level* L = (Level*)h;
  int n = L->n;
  struct Rec { int64_t K, J, I, slot; };
  std::vector<Rec> recs;
  recs.reserve((size_t)(L->E * L->n3));
  for (int64_t e = 0; e < L->E; ++e) {
    int ex, ey, ez; L->elem_coords(e, ex, ey, ez);
    for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
      // reference coordinate in units of 1/(nex p): exact integers for the lattice
      recs.push_back({(int64_t)ez * L->p + c, (int64_t)ey * L->p + b, (int64_t)ex * L->p + a,
                      e * L->n3 + a + n * (b + n * c)});
    }
  }
  std::sort(recs.begin(), recs.end(), [](const Rec& x, const Rec& y) {
    if (x.K != y.K) return x.K < y.K;
    if (x.J != y.J) return x.J < y.J;
    return x.I < y.I;
  });
  int64_t id = -1; int64_t pk = -1, pj = -1, pi = -1;
  for (const Rec& r : recs) {
    if (r.K != pk || r.J != pj || r.I != pi) { ++id; pk = r.K; pj = r.J; pi = r.I; }
    l2g[r.slot] = (int32_t)id;
  }
  return (id + 1 == L->N) ? 0 : 1;
}

// The closed-form lattice numbering used by every other oracle routine (Level::l2g).
int orc_l2g_closed(void* h, int32_t* l2g) {
  Level* L = (Level*)h;
  int n = L->n;
  for (int64_t e = 0; e < L->E; ++e)
    for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
      l2g[e * L->n3 + a + n * (b + n * c)] = (int32_t)L->l2g(e, a, b, c);
  return 0;
}

// Boundary mask by geometry of the reference cube: a node lies on the boundary iff one of its
// reference coordinates is 0 or 1 (exact in lattice units).
int orc_mask(void* h, uint8_t* mask) {
  Level* L = (Level*)h;
  for (int64_t g = 0; g < L->N; ++g) mask[g] = L->boundary(g) ? 1 : 0;
  return 0;
}

int orc_colors(void* h, uint8_t* col) {
  Level* L = (Level*)h;
  for (int64_t e = 0; e < L->E; ++e) {
    int ex, ey, ez; L->elem_coords(e, ex, ey, ez);
    col[e] = (uint8_t)((ex & 1) | ((ey & 1) << 1) | ((ez & 1) << 2));
  }
  return 0;
}

// Geometric factors of element e: G [6][n^3] (00,01,02,11,12,22), detJ [n^3], x [3][n^3].
int orc_geometry(void* h, int64_t e, double* G, double* detJ, double* X) {
  Level* L = (Level*)h;
  if (e < 0 || e >= L->E) return 1;
  element_geometry(*L, e, G, detJ, L->geom_tier);
  if (X) {
    std::vector<double> xs;
    element_nodes(*L, e, xs);
    std::memcpy(X, xs.data(), sizeof(double) * xs.size());
  }
  return 0;
}

// Lazy levels: precompute and keep the geometric factors of the listed elements, so that a
// timed apply over them (bench.py cpu_baseline) measures the operator, not the setup.
int orc_level_cache_elements(void* h, int64_t ne, const int64_t* elems) {
  Level* L = (Level*)h;
  if (L->eager) return 0;
  L->gslot.assign(L->E, -1);
  L->Gcache.assign((size_t)ne * 6 * L->n3, 0.0);
  for (int64_t t = 0; t < ne; ++t) L->gslot[elems[t]] = t;
#pragma omp parallel for schedule(dynamic)
  for (int64_t t = 0; t < ne; ++t)
    element_geometry(*L, elems[t], &L->Gcache[(size_t)t * 6 * L->n3], nullptr, L->geom_tier);
  return 0;
}

int orc_element_matrix(void* h, int64_t e, double* K) {
  Level* L = (Level*)h;
  std::vector<double> buf;
  element_matrix(*L, elem_G(*L, e, buf), K);
  return 0;
}

// Dense assembled A (bc=1) or A_D (bc=0), N x N row-major (tiny meshes only).
int orc_assemble_dense(void* h, int bc, double* A) {
  Level* L = (Level*)h;
  int n = L->n; int64_t n3 = L->n3, N = L->N;
  if (N > 20000) return 1;
  std::fill(A, A + N * N, 0.0);
  std::vector<double> K(n3 * n3), buf;
  for (int64_t e = 0; e < L->E; ++e) {
    element_matrix(*L, elem_G(*L, e, buf), K.data());
    std::vector<int64_t> gl(n3);
    for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
      gl[a + n * (b + n * c)] = L->l2g(e, a, b, c);
    for (int64_t l = 0; l < n3; ++l)
      for (int64_t m = 0; m < n3; ++m) A[gl[l] * N + gl[m]] += K[l * n3 + m];
  }
  if (bc == 0)
    for (int64_t g = 0; g < N; ++g)
      if (L->boundary(g)) {
        for (int64_t m = 0; m < N; ++m) { A[g * N + m] = 0.0; A[m * N + g] = 0.0; }
        A[g * N + g] = 1.0;
      }
  return 0;
}

int orc_apply(void* h, int bc, const double* u, double* v, int tier) {
  apply(*(Level*)h, bc, u, v, tier);
  return 0;
}

// Apply restricted to the elements listed (in order), no boundary handling: the
// element-local O2/O3 results are summed into v (v zeroed first).  Used to time a bounded
// sample of the O2 apply (bench.py cpu_baseline).
int orc_apply_elements(void* h, const double* u, double* v, int64_t ne, const int64_t* elems, int tier) {
  Level* L = (Level*)h;
  int n = L->n; int64_t n3 = L->n3;
  for (int64_t g = 0; g < L->N; ++g) v[g] = 0.0;
  std::vector<double> out((size_t)ne * n3);
#pragma omp parallel
  {
    std::vector<double> ue(n3), gbuf;
#pragma omp for schedule(dynamic)
    for (int64_t t = 0; t < ne; ++t) {
      int64_t e = elems[t];
      for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
        ue[a + n * (b + n * c)] = u[L->l2g(e, a, b, c)];
      const double* G = elem_G(*L, e, gbuf);
      if (tier == 2) element_apply_o2(*L, G, ue.data(), &out[t * n3]);
      else element_apply_o3(*L, G, ue.data(), &out[t * n3]);
    }
  }
  for (int64_t t = 0; t < ne; ++t)
    for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
      v[L->l2g(elems[t], a, b, c)] += out[t * n3 + a + n * (b + n * c)];
  return 0;
}

// Sampled rows of A_D u (bc=0) or A u (bc=1), computed from the <= 8 elements touching each
// row (SURVEY 8(d) "parity sampling").  tier 2 or 3.
int orc_apply_rows(void* h, int bc, const double* u, int64_t nrows, const int64_t* rows,
                   double* out, int tier) {
  Level* L = (Level*)h;
  int n = L->n, p = L->p; int64_t n3 = L->n3;
  std::map<int64_t, int64_t> slot;   // element -> index in elems
  std::vector<int64_t> elems;
  auto cands = [&](int64_t I, int ne, int* c) {
    int k = 0;
    if (I % p == 0 && I > 0) c[k++] = (int)(I / p) - 1;
    if (I / p < ne) c[k++] = (int)(I / p);
    return k;
  };
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t g = rows[r];
    if (bc == 0 && L->boundary(g)) continue;
    int64_t I = g % L->Mx, J = (g / L->Mx) % L->My, K = g / (L->Mx * L->My);
    int cx[2], cy[2], cz[2];
    int nx = cands(I, L->nex, cx), ny = cands(J, L->ney, cy), nz = cands(K, L->nez, cz);
    for (int z = 0; z < nz; ++z) for (int y = 0; y < ny; ++y) for (int x = 0; x < nx; ++x) {
      int64_t e = cx[x] + (int64_t)L->nex * (cy[y] + (int64_t)L->ney * cz[z]);
      if (!slot.count(e)) { slot[e] = (int64_t)elems.size(); elems.push_back(e); }
    }
  }
  std::vector<double> ev(elems.size() * n3);
#pragma omp parallel
  {
    std::vector<double> ue(n3), gbuf;
#pragma omp for schedule(dynamic)
    for (int64_t t = 0; t < (int64_t)elems.size(); ++t) {
      int64_t e = elems[t];
      for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
        int64_t gg = L->l2g(e, a, b, c);
        ue[a + n * (b + n * c)] = (bc == 0 && L->boundary(gg)) ? 0.0 : u[gg];
      }
      const double* G = elem_G(*L, e, gbuf);
      if (tier == 2) element_apply_o2(*L, G, ue.data(), &ev[t * n3]);
      else element_apply_o3(*L, G, ue.data(), &ev[t * n3]);
    }
  }
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t g = rows[r];
    if (bc == 0 && L->boundary(g)) { out[r] = u[g]; continue; }
    int64_t I = g % L->Mx, J = (g / L->Mx) % L->My, K = g / (L->Mx * L->My);
    int cx[2], cy[2], cz[2];
    int nx = cands(I, L->nex, cx), ny = cands(J, L->ney, cy), nz = cands(K, L->nez, cz);
    double s = 0.0;
    for (int z = 0; z < nz; ++z) for (int y = 0; y < ny; ++y) for (int x = 0; x < nx; ++x) {
      int64_t e = cx[x] + (int64_t)L->nex * (cy[y] + (int64_t)L->ney * cz[z]);
      int a = (int)(I - (int64_t)cx[x] * p), b = (int)(J - (int64_t)cy[y] * p), c = (int)(K - (int64_t)cz[z] * p);
      s += ev[slot[e] * n3 + a + n * (b + n * c)];
    }
    out[r] = s;
  }
  return 0;
}

int orc_diag(void* h, int bc, double* d) {
  compute_diag(*(Level*)h, bc, d);
  return 0;
}

double orc_lambda_max(void* h, int iters, uint64_t seed) {
  return lambda_max(*(Level*)h, iters, seed, nullptr);
}

int orc_cheb(void* h, const double* b, double* x, int K, double lo, double hi) {
  chebyshev(*(Level*)h, b, x, K, lo, hi, nullptr);
  return 0;
}

double orc_lambda_arnoldi(void* h, int m, uint64_t seed) {
  return lambda_arnoldi(*(Level*)h, m, seed, nullptr);
}

int orc_jacobi(void* h, const double* b, double* x, int steps, double omega) {
  jacobi(*(Level*)h, b, x, steps, omega, nullptr);
  return 0;
}

int orc_pair_kind(void* hc, void* hf) { return pair_kind(*(Level*)hc, *(Level*)hf); }

int orc_prolong(void* hc, void* hf, const double* uc, double* uf) {
  Level* C = (Level*)hc; Level* F = (Level*)hf;
  if (!pair_kind(*C, *F)) return 5;   // p pair or h pair
  transfer_prolong(*C, *F, uc, uf);
  return 0;
}

int orc_restrict(void* hc, void* hf, const double* rf, double* rc) {
  Level* C = (Level*)hc; Level* F = (Level*)hf;
  if (!pair_kind(*C, *F)) return 5;
  transfer_restrict(*C, *F, rf, rc);
  return 0;
}

// Load vector of the manufactured solution u* = sin(pi x) sin(pi y) sin(pi z) (SURVEY 8(c)
// step 12): f = -div(mu grad u*) = 3 pi^2 mu u* - grad mu . grad u*, collocated quadrature
// b_g = (1 - bnd_g) sum_{(e,q) -> g} w_q detJ_q f(x_q)  (A9).  rhs_id 1.
int orc_load_vector(void* h, int rhs_id, double* f) {
  Level* L = (Level*)h;
  if (rhs_id != 1) return 1;
  int n = L->n; int64_t n3 = L->n3;
  for (int64_t g = 0; g < L->N; ++g) f[g] = 0.0;
  for (int col = 0; col < 8; ++col) {
    const std::vector<int64_t>& els = L->colour_elems[col];
#pragma omp parallel
    {
      std::vector<double> G(6 * n3), dJ(n3), X;
#pragma omp for schedule(static)
      for (int64_t t = 0; t < (int64_t)els.size(); ++t) {
        int64_t e = els[t];
        element_geometry(*L, e, G.data(), dJ.data(), L->geom_tier);
        element_nodes(*L, e, X);
        for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
          int64_t q = a + n * (b + n * c);
          double xq[3] = {X[q], X[n3 + q], X[2 * n3 + q]};
          if (L->B.quad == 1) quad_point(*L, X, a, b, c, xq);
          double x = xq[0], y = xq[1], z = xq[2];
          double us = std::sin(kPi * x) * std::sin(kPi * y) * std::sin(kPi * z);
          double gu[3] = {kPi * std::cos(kPi * x) * std::sin(kPi * y) * std::sin(kPi * z),
                          kPi * std::sin(kPi * x) * std::cos(kPi * y) * std::sin(kPi * z),
                          kPi * std::sin(kPi * x) * std::sin(kPi * y) * std::cos(kPi * z)};
          double gm[3];
          coeff_grad(L->coeff, L->c0, L->c1, x, y, z, gm);
          double mu = coeff_mu(L->coeff, L->c0, L->c1, x, y, z);
          double fx = 3.0 * kPi * kPi * mu * us - (gm[0] * gu[0] + gm[1] * gu[1] + gm[2] * gu[2]);
          const double wq = L->B.qw[a] * L->B.qw[b] * L->B.qw[c] * dJ[q] * fx;
          if (L->B.quad == 0) { f[L->l2g(e, a, b, c)] += wq; continue; }
          for (int cc = 0; cc < n; ++cc) for (int bb = 0; bb < n; ++bb) for (int aa = 0; aa < n; ++aa)   // phi_l(x_q)
            f[L->l2g(e, aa, bb, cc)] += L->B.L[a * n + aa] * L->B.L[b * n + bb] * L->B.L[c * n + cc] * wq;
        }
      }
    }
  }
  for (int64_t g = 0; g < L->N; ++g) if (L->boundary(g)) f[g] = 0.0;
  return 0;
}

// Exact solution u* at the physical nodes (for the MMS convergence pin).
int orc_exact_solution(void* h, double* u) {
  Level* L = (Level*)h;
  int n = L->n; int64_t n3 = L->n3;
  std::vector<double> X;
  for (int64_t e = 0; e < L->E; ++e) {
    element_nodes(*L, e, X);
    for (int c = 0; c < n; ++c) for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
      int64_t q = a + n * (b + n * c);
      u[L->l2g(e, a, b, c)] = std::sin(kPi * X[q]) * std::sin(kPi * X[n3 + q]) * std::sin(kPi * X[2 * n3 + q]);
    }
  }
  return 0;
}

// Plain CG on a dense SPD matrix (pin S:433); M = I.  Returns iterations in *iters.
int orc_cg_dense(int n, const double* A, const double* b, double* x, double rtol, int maxit, int* iters) {
  std::vector<double> r(b, b + n), p(b, b + n), Ap(n);
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  double rr = 0.0; for (int i = 0; i < n; ++i) rr += r[i] * r[i];
  double r0 = std::sqrt(rr);
  int it = 0;
  while (it < maxit && std::sqrt(rr) > rtol * r0) {
    for (int i = 0; i < n; ++i) { double s = 0; for (int j = 0; j < n; ++j) s += A[i * n + j] * p[j]; Ap[i] = s; }
    double pAp = 0; for (int i = 0; i < n; ++i) pAp += p[i] * Ap[i];
    if (pAp <= 0.0) { *iters = it; return 6; }
    double alpha = rr / pAp;
    for (int i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; }
    double rn = 0; for (int i = 0; i < n; ++i) rn += r[i] * r[i];
    for (int i = 0; i < n; ++i) p[i] = r[i] + (rn / rr) * p[i];
    rr = rn; ++it;
  }
  *iters = it;
  return 0;
}

// coarsen 0: p-multigrid hierarchy p, p/2, ..., 1 on one element grid (R20), followed by
// h_levels geometric coarsenings of the p = 1 mesh (ne -> ne/2 -> ...; NEXT-1).
// coarsen 1: high-order h-multigrid (NEXT-4): order p on meshes ne, ne/2, ..., ne/2^h_levels
// ("three levels with 8x8x8, 4x4x4 and 2x2x2 elements"), any p.
// smoother 0: Chebyshev-Jacobi of degree K; 1: damped point Jacobi (omega), one step per smoothing
// application.  lambda_method 0: power iteration (R9), 1: Arnoldi (R26), power_iters steps.
void* orc_hier_create3(int nex, int ney, int nez, int p, int warp, double amp, int coeff, double c0,
                       double c1, int nu_pre, int nu_post, int K, double lo_frac, double hi_frac,
                       int power_iters, uint64_t seed, double coarse_rtol, int coarse_maxit,
                       int geom_tier, int tier, int smoother, double omega, int lambda_method, int h_levels,
                       int coarsen, int* status) {
  *status = 0;
  const int p_levels_to = (coarsen == 1) ? p : 1;   // orders kept: p, ..., p_levels_to
  for (int q = p; q > p_levels_to; q /= 2)
    if (q % 2) { *status = 5; return nullptr; }
  for (int j = 0; j < h_levels; ++j)
    if (((nex >> j) % 2) || ((ney >> j) % 2) || ((nez >> j) % 2)) { *status = 5; return nullptr; }
  Hier* H = new Hier();
  H->nu_pre = nu_pre; H->nu_post = nu_post; H->K = K; H->lo_frac = lo_frac; H->hi_frac = hi_frac;
  H->power_iters = power_iters; H->seed = seed; H->coarse_rtol = coarse_rtol; H->coarse_maxit = coarse_maxit;
  H->smoother = smoother; H->omega = omega; H->lambda_method = lambda_method;
  for (int q = p; q >= p_levels_to; q /= 2) {
    Level* L = (Level*)orc_level_create(nex, ney, nez, q, warp, amp, coeff, c0, c1, 1, geom_tier, tier);
    if (!L) { *status = 1; return H; }
    if (L->status) *status = L->status;
    H->lv.push_back(L);
    if (q == p_levels_to) break;
  }
  for (int j = 1; j <= h_levels; ++j) {
    Level* L = (Level*)orc_level_create(nex >> j, ney >> j, nez >> j, p_levels_to, warp, amp, coeff, c0, c1, 1,
                                        geom_tier, tier);
    if (!L) { *status = 1; return H; }
    if (L->status) *status = L->status;
    H->lv.push_back(L);
  }
  H->lam.assign(H->lv.size(), 0.0);
  for (size_t l = 0; l + 1 < H->lv.size(); ++l)
    H->lam[l] = lambda_method == 1 ? lambda_arnoldi(*H->lv[l], power_iters, seed, nullptr)
                                   : lambda_max(*H->lv[l], power_iters, seed, nullptr);
  return H;
}

void* orc_hier_create2(int nex, int ney, int nez, int p, int warp, double amp, int coeff, double c0,
                       double c1, int nu_pre, int nu_post, int K, double lo_frac, double hi_frac,
                       int power_iters, uint64_t seed, double coarse_rtol, int coarse_maxit,
                       int geom_tier, int tier, int smoother, double omega, int lambda_method, int h_levels,
                       int* status) {
  return orc_hier_create3(nex, ney, nez, p, warp, amp, coeff, c0, c1, nu_pre, nu_post, K, lo_frac, hi_frac,
                          power_iters, seed, coarse_rtol, coarse_maxit, geom_tier, tier, smoother, omega,
                          lambda_method, h_levels, 0, status);
}

void* orc_hier_create(int nex, int ney, int nez, int p, int warp, double amp, int coeff, double c0,
                      double c1, int nu_pre, int nu_post, int K, double lo_frac, double hi_frac,
                      int power_iters, uint64_t seed, double coarse_rtol, int coarse_maxit,
                      int geom_tier, int tier, int* status) {
  return orc_hier_create2(nex, ney, nez, p, warp, amp, coeff, c0, c1, nu_pre, nu_post, K, lo_frac, hi_frac,
                          power_iters, seed, coarse_rtol, coarse_maxit, geom_tier, tier, 0, 2.0 / 3.0, 0, 0,
                          status);
}

void orc_hier_destroy(void* h) {
  Hier* H = (Hier*)h;
  for (Level* L : H->lv) delete L;
  delete H;
}

int orc_hier_nlevels(void* h) { return (int)((Hier*)h)->lv.size(); }
void* orc_hier_level(void* h, int l) { return ((Hier*)h)->lv[l]; }
double orc_hier_lambda(void* h, int l) { return ((Hier*)h)->lam[l]; }
int64_t orc_hier_fine_applies(void* h) { return ((Hier*)h)->fine_applies; }
int64_t orc_hier_coarse_iters(void* h) { return ((Hier*)h)->coarse_iters_last; }

int orc_vcycle(void* h, const double* b, double* x) {
  return vcycle(*(Hier*)h, 0, b, x);
}

// mode 0: MG as solver x <- x + V(b - A x); mode 1: MG-preconditioned CG (Algorithm 1,
// P:973-991).  x0 = 0 (R14); stop at ||r||_2 <= rtol ||r0||_2.
// Divergence (||r|| > 10 ||r0||) stops with converged = 0.
int orc_solve(void* h, int mode, const double* b, double* x, double rtol, int maxit,
              int* iters_out, int* converged, double* r0n, double* rn, double* hist, int hist_cap,
              int64_t* fine_applies) {
  return solve_impl((Hier*)h, mode, b, x, rtol, maxit, iters_out, converged, r0n, rn, hist, hist_cap, fine_applies);
}

/* ---------------------------------------------------------------- NEXT-2: 2-D C ABI (orc2_*) */
void* orc2_level_create(int nex, int ney, int p, int warp, double amp, int coeff, double c0, double c1) {
  if (p < 1 || p > 16 || nex < 1 || ney < 1) return nullptr;
  Level2* L = new Level2();
  L->nex = nex; L->ney = ney; L->p = p; L->n = p + 1;
  L->warp = warp; L->amp = amp; L->coeff = coeff; L->c0 = c0; L->c1 = c1;
  L->E = (int64_t)nex * ney;
  L->Mx = (int64_t)nex * p + 1; L->My = (int64_t)ney * p + 1;
  L->N = L->Mx * L->My;
  L->n2 = (int64_t)L->n * L->n;
  L->B.build(p, g_quad);
  L->colour_elems.assign(4, {});
  for (int64_t e = 0; e < L->E; ++e) {
    int ex, ey; L->elem_coords(e, ex, ey);
    L->colour_elems[(ex & 1) | ((ey & 1) << 1)].push_back(e);
  }
  L->G.resize((size_t)L->E * 3 * L->n2);
  L->detJ.resize((size_t)L->E * L->n2);
  double mind = 1e300;
  for (int64_t e = 0; e < L->E; ++e)
    mind = std::min(mind, element_geometry2(*L, e, &L->G[(size_t)e * 3 * L->n2], &L->detJ[(size_t)e * L->n2]));
  L->min_detj = mind;
  if (!(mind > 0.0)) L->status = 4;
  return L;
}
void orc2_level_destroy(void* h) { delete (Level2*)h; }
int orc2_level_status(void* h) { return ((Level2*)h)->status; }
int64_t orc2_level_ndofs(void* h) { return ((Level2*)h)->N; }
int orc2_mask(void* h, uint8_t* mask) {
  Level2* L = (Level2*)h;
  for (int64_t g = 0; g < L->N; ++g) mask[g] = L->boundary(g) ? 1 : 0;
  return 0;
}
int orc2_geometry(void* h, int64_t e, double* G) {
  Level2* L = (Level2*)h;
  for (int64_t i = 0; i < 3 * L->n2; ++i) G[i] = L->G[(size_t)e * 3 * L->n2 + i];
  return 0;
}
int orc2_element_matrix(void* h, int64_t e, double* K) {
  Level2* L = (Level2*)h;
  element_matrix2(*L, &L->G[(size_t)e * 3 * L->n2], K);
  return 0;
}
// Dense A_D (bc 0) or A (bc 1) assembled from the element matrices (O1), small meshes only.
int orc2_assemble_dense(void* h, int bc, double* A) {
  Level2* L = (Level2*)h;
  const int n = L->n; const int64_t n2 = L->n2, N = L->N;
  for (int64_t i = 0; i < N * N; ++i) A[i] = 0.0;
  std::vector<double> K(n2 * n2);
  for (int64_t e = 0; e < L->E; ++e) {
    element_matrix2(*L, &L->G[(size_t)e * 3 * n2], K.data());
    for (int64_t l = 0; l < n2; ++l)
      for (int64_t m = 0; m < n2; ++m) A[L->l2g(e, (int)(l % n), (int)(l / n)) * N + L->l2g(e, (int)(m % n), (int)(m / n))] += K[l * n2 + m];
  }
  if (bc == 0)
    for (int64_t g = 0; g < N; ++g)
      if (L->boundary(g)) {
        for (int64_t k = 0; k < N; ++k) { A[g * N + k] = 0.0; A[k * N + g] = 0.0; }
        A[g * N + g] = 1.0;
      }
  return 0;
}
int orc2_apply(void* h, int bc, const double* u, double* v) { apply(*(Level2*)h, bc, u, v, 2); return 0; }
int orc2_diag(void* h, int bc, double* d) { compute_diag(*(Level2*)h, bc, d); return 0; }
double orc2_lambda_max(void* h, int iters, uint64_t seed) { return lambda_max(*(Level2*)h, iters, seed, nullptr); }
double orc2_lambda_arnoldi(void* h, int m, uint64_t seed) { return lambda_arnoldi(*(Level2*)h, m, seed, nullptr); }
int orc2_cheb(void* h, const double* b, double* x, int K, double lo, double hi) {
  chebyshev(*(Level2*)h, b, x, K, lo, hi, nullptr);
  return 0;
}
int orc2_jacobi(void* h, const double* b, double* x, int steps, double omega) {
  jacobi(*(Level2*)h, b, x, steps, omega, nullptr);
  return 0;
}
int orc2_prolong(void* hc, void* hf, const double* uc, double* uf) {
  Level2 *C = (Level2*)hc, *F = (Level2*)hf;
  if (!pair_kind(*C, *F)) return 5;
  transfer_prolong(*C, *F, uc, uf);
  return 0;
}
int orc2_restrict(void* hc, void* hf, const double* rf, double* rc) {
  Level2 *C = (Level2*)hc, *F = (Level2*)hf;
  if (!pair_kind(*C, *F)) return 5;
  transfer_restrict(*C, *F, rf, rc);
  return 0;
}
// Manufactured solution u* = sin(pi x) sin(pi y): f = -div(mu grad u*) = 2 pi^2 mu u* - grad mu . grad u*,
// b_l = (1 - bnd) sum_{e, q} phi_l(x_q) w_q detJ_q f(x_q); rhs_id 1.
int orc2_load_vector(void* h, int rhs_id, double* f) {
  Level2* L = (Level2*)h;
  if (rhs_id != 1) return 1;
  const int n = L->n; const int64_t n2 = L->n2;
  for (int64_t g = 0; g < L->N; ++g) f[g] = 0.0;
  std::vector<double> X;
  for (int64_t e = 0; e < L->E; ++e) {
    element_nodes2(*L, e, X);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double x = 0.0, y = 0.0;
        for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a) {
          const double ph = L->B.L[i * n + a] * L->B.L[j * n + b];
          x += ph * X[a + n * b]; y += ph * X[n2 + a + n * b];
        }
        const double us = std::sin(kPi * x) * std::sin(kPi * y);
        const double gu[2] = {kPi * std::cos(kPi * x) * std::sin(kPi * y), kPi * std::sin(kPi * x) * std::cos(kPi * y)};
        double gm[2];
        coeff_grad2(L->coeff, L->c0, L->c1, x, y, gm);
        const double fx = 2.0 * kPi * kPi * coeff_mu2(L->coeff, L->c0, L->c1, x, y) * us - (gm[0] * gu[0] + gm[1] * gu[1]);
        const double wq = L->B.qw[i] * L->B.qw[j] * L->detJ[(size_t)e * n2 + i + n * j] * fx;
        for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
          f[L->l2g(e, a, b)] += L->B.L[i * n + a] * L->B.L[j * n + b] * wq;
      }
  }
  for (int64_t g = 0; g < L->N; ++g) if (L->boundary(g)) f[g] = 0.0;
  return 0;
}
int orc2_exact_solution(void* h, double* u) {
  Level2* L = (Level2*)h;
  const int n = L->n;
  std::vector<double> X;
  for (int64_t e = 0; e < L->E; ++e) {
    element_nodes2(*L, e, X);
    for (int b = 0; b < n; ++b) for (int a = 0; a < n; ++a)
      u[L->l2g(e, a, b)] = std::sin(kPi * X[a + n * b]) * std::sin(kPi * X[L->n2 + a + n * b]);
  }
  return 0;
}
// Hierarchy (as orc_hier_create3): coarsen 0: p, p/2, ..., 1 then h_levels meshes at p = 1;
// coarsen 1: order p on ne, ne/2, ..., ne/2^h_levels ("32x32, 16x16 and 8x8").
void* orc2_hier_create(int nex, int ney, int p, int warp, double amp, int coeff, double c0, double c1, int nu_pre,
                       int nu_post, int K, double lo_frac, double hi_frac, int power_iters, uint64_t seed,
                       double coarse_rtol, int coarse_maxit, int smoother, double omega, int lambda_method,
                       int h_levels, int coarsen, int* status) {
  *status = 0;
  const int pmin = (coarsen == 1) ? p : 1;
  for (int q = p; q > pmin; q /= 2)
    if (q % 2) { *status = 5; return nullptr; }
  for (int j = 0; j < h_levels; ++j)
    if (((nex >> j) % 2) || ((ney >> j) % 2)) { *status = 5; return nullptr; }
  Hier2* H = new Hier2();
  H->nu_pre = nu_pre; H->nu_post = nu_post; H->K = K; H->lo_frac = lo_frac; H->hi_frac = hi_frac;
  H->power_iters = power_iters; H->seed = seed; H->coarse_rtol = coarse_rtol; H->coarse_maxit = coarse_maxit;
  H->smoother = smoother; H->omega = omega; H->lambda_method = lambda_method;
  for (int q = p; q >= pmin; q /= 2) {
    H->lv.push_back((Level2*)orc2_level_create(nex, ney, q, warp, amp, coeff, c0, c1));
    if (q == pmin) break;
  }
  for (int j = 1; j <= h_levels; ++j)
    H->lv.push_back((Level2*)orc2_level_create(nex >> j, ney >> j, pmin, warp, amp, coeff, c0, c1));
  for (Level2* L : H->lv) if (L->status) *status = L->status;
  H->lam.assign(H->lv.size(), 0.0);
  for (size_t l = 0; l + 1 < H->lv.size(); ++l)
    H->lam[l] = lambda_method == 1 ? lambda_arnoldi(*H->lv[l], power_iters, seed, nullptr)
                                   : lambda_max(*H->lv[l], power_iters, seed, nullptr);
  return H;
}
void orc2_hier_destroy(void* h) {
  Hier2* H = (Hier2*)h;
  for (Level2* L : H->lv) delete L;
  delete H;
}
int orc2_hier_nlevels(void* h) { return (int)((Hier2*)h)->lv.size(); }
void* orc2_hier_level(void* h, int l) { return ((Hier2*)h)->lv[l]; }
double orc2_hier_lambda(void* h, int l) { return ((Hier2*)h)->lam[l]; }
int orc2_vcycle(void* h, const double* b, double* x) { return vcycle(*(Hier2*)h, 0, b, x); }
int orc2_solve(void* h, int mode, const double* b, double* x, double rtol, int maxit, int* iters_out, int* converged,
               double* r0n, double* rn, double* hist, int hist_cap, int64_t* fine_applies) {
  return solve_impl((Hier2*)h, mode, b, x, rtol, maxit, iters_out, converged, r0n, rn, hist, hist_cap, fine_applies);
}

}  // extern "C"

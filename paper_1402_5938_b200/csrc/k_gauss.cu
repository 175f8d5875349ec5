// Gauss-Legendre quadrature variant of the operator ("The Jacobians for
// this transformation are computed at every quadrature point, and Gauss quadrature is used to
// numerically approximate integrals").  The basis stays the nodal LGL basis of order p; the
// quadrature uses n = p + 1 Gauss-Legendre points per direction (exact for degree 2p + 1, so the
// stiffness of affine elements is integrated exactly).  Tables (host, per order):
//   B[i][a]  = ell_a(xi_i)     nodal basis at the Gauss points          (interpolation)
//   DB[i][a] = ell_a'(xi_i)    its derivative (geometry)
//   DG[i][m] = ell^G_m'(xi_i)  derivative matrix of the Lagrange basis on the Gauss points
// Apply per element (same structure as the collocated operator on the Gauss grid, wrapped in
// interpolations): u_q = (B x B x B) u_e; g = (DG x I x I, I x DG x I, I x I x DG) u_q (exact: u_q
// represents the same degree-p polynomial); w = G_q g; v_q = DG^T contractions of w;
// v_e = (B^T x B^T x B^T) v_q; scatter.  G_q = wG_i wG_j wG_k mu(x(xi_q)) detJ_q J_q^{-1} J_q^{-T}
// with J and x from the isoparametric map evaluated at the Gauss points.
#include <cmath>
#include <cstdlib>

#include "k_common.cuh"

namespace sfmg {

constexpr int qOffset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += (q + 1) * (q + 1);
  return s;
}
constexpr int qvOffset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += q + 1;
  return s;
}
__constant__ double c_qB[qOffset(kMaxOrder + 1)];
__constant__ double c_qDB[qOffset(kMaxOrder + 1)];
__constant__ double c_qDG[qOffset(kMaxOrder + 1)];
// Even-odd forms of B, DB, B^T, DB^T for even orders 4..16 (k_apply_gauss_v2): B is centro-symmetric
// (B[n-1-i][n-1-a] = B[i][a]), DB centro-antisymmetric, so a line product splits into an even and an
// odd half of c = p/2 terms each.  Per set: Me[c][c], Mo[c][c], M[i][c] (c), M[c][m] (c), M[c][c].
constexpr int geoSize(int P) { return 2 * (P / 2) * (P / 2) + 2 * (P / 2) + 1; }
constexpr int geoOffset(int P) {
  int s = 0;
  for (int q = 4; q < P; q += 2) s += 4 * geoSize(q);
  return s;
}
constexpr int kGaussV2MaxP = 16;
__constant__ double c_gEO[geoOffset(kGaussV2MaxP + 2)];
__constant__ double c_qw[qvOffset(kMaxOrder + 1)];   // Gauss weights
__constant__ double c_qxn[qvOffset(kMaxOrder + 1)];  // LGL nodes (node positions)

// ---------------------------------------------------------------------------- host tables

// Gauss-Legendre points (roots of P_n) and weights 2 / ((1 - x^2) P_n'(x)^2): Newton's method on
// the three-term recurrence from the Chebyshev-like guesses cos(pi (i + 3/4) / (n + 1/2)).
static void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (n - 1 - i + 0.75) / (n + 0.5));   // ascending order
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      const double pn = (n == 0) ? 1.0 : p1, pm = (n == 0) ? 0.0 : p0;
      dp = n * (t * pn - pm) / (t * t - 1.0);
      const double dt = pn / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    double p0 = 1.0, p1 = t;
    for (int k = 2; k <= n; ++k) {
      const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = n * (t * p1 - p0) / (t * t - 1.0);
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
  for (int i = 0; i < n / 2; ++i) {   // exact symmetry
    const double a = 0.5 * (x[n - 1 - i] - x[i]), b = 0.5 * (w[i] + w[n - 1 - i]);
    x[i] = -a;
    x[n - 1 - i] = a;
    w[i] = w[n - 1 - i] = b;
  }
  if (n % 2) x[n / 2] = 0.0;
}

// Lagrange cardinal ell_a on nodes xs at t (barycentric weights), and its derivative.
static double lag_val(const std::vector<double>& xs, int a, double t) {
  double v = 1.0;
  for (size_t k = 0; k < xs.size(); ++k)
    if ((int)k != a) v *= (t - xs[k]) / (xs[a] - xs[k]);
  return v;
}
static double lag_der(const std::vector<double>& xs, int a, double t) {
  double s = 0.0;
  for (size_t j = 0; j < xs.size(); ++j) {
    if ((int)j == a) continue;
    double v = 1.0 / (xs[a] - xs[j]);
    for (size_t k = 0; k < xs.size(); ++k)
      if ((int)k != a && k != j) v *= (t - xs[k]) / (xs[a] - xs[k]);
    s += v;
  }
  return s;
}

// 1-D tables of one order for the 2-D kernels (k_2d.cu): LGL nodes, and the basis / derivative at the
// quadrature points with their weights: quad 0 collocated LGL (B = I, DB = D, w_LGL), quad 1 Gauss.
void quad_tables_1d(int p, int quad, std::vector<double>& xn, std::vector<double>& B, std::vector<double>& DB,
                    std::vector<double>& qw) {
  const int n = p + 1;
  Basis1D L = make_basis(p);
  xn = L.x;
  B.assign(n * n, 0.0);
  DB.assign(n * n, 0.0);
  if (quad == 0) {
    for (int i = 0; i < n; ++i) B[i * n + i] = 1.0;
    DB = L.D;
    qw = L.w;
    return;
  }
  std::vector<double> gx;
  gauss_rule(n, gx, qw);
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < n; ++a) {
      B[i * n + a] = lag_val(L.x, a, gx[i]);
      DB[i * n + a] = lag_der(L.x, a, gx[i]);
    }
}

static OncePerDevice g_gauss_uploaded[kMaxOrder + 1];

cudaError_t upload_gauss_tables(int p) {
  if (p < 1 || p > kMaxOrder) return cudaErrorInvalidValue;
  return g_gauss_uploaded[p].run([&]() -> cudaError_t {
  const int n = p + 1;
  Basis1D L = make_basis(p);
  std::vector<double> gx, gw;
  gauss_rule(n, gx, gw);
  std::vector<double> B(n * n), DB(n * n), DG(n * n);
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < n; ++a) {
      B[i * n + a] = lag_val(L.x, a, gx[i]);
      DB[i * n + a] = lag_der(L.x, a, gx[i]);
      DG[i * n + a] = lag_der(gx, a, gx[i]);
    }
  const size_t mo = sizeof(double) * qOffset(p), vo = sizeof(double) * qvOffset(p);
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(c_qB, B.data(), sizeof(double) * n * n, mo))) return e;
  if ((e = cudaMemcpyToSymbol(c_qDB, DB.data(), sizeof(double) * n * n, mo))) return e;
  if ((e = cudaMemcpyToSymbol(c_qDG, DG.data(), sizeof(double) * n * n, mo))) return e;
  if (p % 2 == 0 && p >= 4 && p <= kGaussV2MaxP) {
    const int c = p / 2;
    std::vector<double> tab(4 * geoSize(p));
    for (int set = 0; set < 4; ++set) {
      auto M = [&](int i, int m2) {
        switch (set) {
          case 0: return B[i * n + m2];
          case 1: return DB[i * n + m2];
          case 2: return B[m2 * n + i];
          default: return DB[m2 * n + i];
        }
      };
      double* t = tab.data() + set * geoSize(p);
      for (int i = 0; i < c; ++i)
        for (int m2 = 0; m2 < c; ++m2) {
          t[i * c + m2] = 0.5 * (M(i, m2) + M(i, n - 1 - m2));
          t[c * c + i * c + m2] = 0.5 * (M(i, m2) - M(i, n - 1 - m2));
        }
      for (int i = 0; i < c; ++i) t[2 * c * c + i] = M(i, c);
      for (int m2 = 0; m2 < c; ++m2) t[2 * c * c + c + m2] = M(c, m2);
      t[2 * c * c + 2 * c] = M(c, c);
    }
    if ((e = cudaMemcpyToSymbol(c_gEO, tab.data(), sizeof(double) * tab.size(), sizeof(double) * geoOffset(p)))) return e;
  }
  if ((e = cudaMemcpyToSymbol(c_qw, gw.data(), sizeof(double) * n, vo))) return e;
  if ((e = cudaMemcpyToSymbol(c_qxn, L.x.data(), sizeof(double) * n, vo))) return e;
  return cudaSuccess;
  });
}

template <int P> __device__ __forceinline__ double qB(int i, int a) { return c_qB[qOffset(P) + i * (P + 1) + a]; }
template <int P> __device__ __forceinline__ double qDG(int i, int a) { return c_qDG[qOffset(P) + i * (P + 1) + a]; }

// Element geometry at the Gauss points into smem tables: per point J (9), x (3), from the nodal
// positions X[3][n^3] (smem) and the B / DB tables (smem copies sB, sDB).
template <int P>
__device__ __forceinline__ void gauss_jacobian(const double* X, const double* sB, const double* sDB, int i, int j, int k,
                                               double J[3][3], double xq[3]) {
  constexpr int N = P + 1, N3 = N * N * N;
#pragma unroll
  for (int al = 0; al < 3; ++al) { J[al][0] = J[al][1] = J[al][2] = 0.0; xq[al] = 0.0; }
  for (int c = 0; c < N; ++c) {
    const double Bk = sB[k * N + c], Dk = sDB[k * N + c];
    for (int b = 0; b < N; ++b) {
      const double Bj = sB[j * N + b], Dj = sDB[j * N + b];
      const double bjk = Bj * Bk, djk = Dj * Bk, bjdk = Bj * Dk;
      for (int a = 0; a < N; ++a) {
        const double Bi = sB[i * N + a], Di = sDB[i * N + a];
        const int l = a + N * (b + N * c);
        const double p0 = Di * bjk, p1 = Bi * djk, p2 = Bi * bjdk, ph = Bi * bjk;
#pragma unroll
        for (int al = 0; al < 3; ++al) {
          const double x = X[al * N3 + l];
          J[al][0] = fma(x, p0, J[al][0]);
          J[al][1] = fma(x, p1, J[al][1]);
          J[al][2] = fma(x, p2, J[al][2]);
          xq[al] = fma(x, ph, xq[al]);
        }
      }
    }
  }
}

template <int P>
__device__ __forceinline__ void load_tables_and_nodes(const MeshDev& m, long long e, double* X, double* sB, double* sDB) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  for (int t = threadIdx.x; t < N2; t += blockDim.x) {
    sB[t] = c_qB[qOffset(P) + t];
    sDB[t] = c_qDB[qOffset(P) + t];
  }
  int ex, ey, ez;
  elem_coords(m, e, ex, ey, ez);
  const double* xn = c_qxn + qvOffset(P);
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int a = l % N, b = (l / N) % N, c = l / N2;
    double x[3];
    node_pos<P>(m, xn, ex, ey, ez, a, b, c, x);
    X[l] = x[0];
    X[N3 + l] = x[1];
    X[2 * N3 + l] = x[2];
  }
}

// ---------------------------------------------------------------------------- geometry

template <int P>
__global__ void __launch_bounds__(256) k_geometry_gauss(MeshDev m, double* __restrict__ G, int* bad) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  extern __shared__ double gsm[];
  double* X = gsm;              // [3][N3]
  double* sB = X + 3 * N3;      // [N2]
  double* sDB = sB + N2;        // [N2]
  const double* w = c_qw + qvOffset(P);
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    __syncthreads();
    load_tables_and_nodes<P>(m, e, X, sB, sDB);
    __syncthreads();
    for (int q = threadIdx.x; q < N3; q += blockDim.x) {
      const int i = q % N, j = (q / N) % N, k = q / N2;
      double J[3][3], xq[3];
      gauss_jacobian<P>(X, sB, sDB, i, j, k, J, xq);
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      if (!(det > 0.0)) atomicAdd(bad, 1);
      const double id = 1.0 / det;
      double Ji[3][3];
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
      const double s = w[i] * w[j] * w[k] * coeff_mu(m, xq[0], xq[1], xq[2]) * det;
      const int comp[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const int a = comp[c][0], b = comp[c][1];
        G[GLayout<P>::off(e, c, i + N * j, k)] = s * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
      }
    }
  }
}

// ---------------------------------------------------------------------------- apply

// out = M L on one line, M[i][m] = B (T = false) or its transpose (T = true), DG likewise.
template <int P, bool T>
__device__ __forceinline__ void line_B(const double (&L)[P + 1], double (&out)[P + 1]) {
  constexpr int N = P + 1;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < N; ++m) s = fma(T ? qB<P>(m, i) : qB<P>(i, m), L[m], s);
    out[i] = s;
  }
}
template <int P, bool T>
__device__ __forceinline__ void line_DG(const double (&L)[P + 1], double (&out)[P + 1]) {
  constexpr int N = P + 1;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < N; ++m) s = fma(T ? qDG<P>(m, i) : qDG<P>(i, m), L[m], s);
    out[i] = s;
  }
}

template <int P>
struct GaussCfg {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr int EPB = 128 / N2 > 0 ? 128 / N2 : 1;
  static constexpr int THREADS = EPB * N2;
  static constexpr size_t SMEM = sizeof(double) * 3 * N3 * EPB;
};

// L2 prefetch (TMA bulk, evict-first policy: the factors are read once) of one group's factors and
// a group's u columns, issued one group ahead so that the pointwise pass and the gather of the next
// group hit L2 (the collocated kernel's scheme, k_operator.cu).
__device__ __forceinline__ void gauss_prefetch_l2(const void* src, unsigned bytes) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (unsigned o = 0; o < bytes; o += 65536u)
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"((const char*)src + o),
                 "r"(bytes - o < 65536u ? bytes - o : 65536u), "l"(pol)
                 : "memory");
}

// Block = EPB elements x n^2 threads; thread (t0, t1) owns one line per pass (see file header).
template <int P, bool DIR>
__global__ void __launch_bounds__(GaussCfg<P>::THREADS) k_apply_gauss(MeshDev m, const double* __restrict__ G,
                                                                      const double* __restrict__ u,
                                                                      double* __restrict__ v) {
  using C = GaussCfg<P>;
  constexpr int N = C::N, N2 = C::N2, N3 = C::N3;
  extern __shared__ double asm_[];
  const int le = threadIdx.x / N2, t = threadIdx.x - le * N2, t0 = t % N, t1 = t / N;
  double* A = asm_ + le * 3 * N3;
  double* Bb = A + N3;
  double* Cc = Bb + N3;
  const long long sxy = (long long)m.Mx * m.My;
  const long long ngroups = (m.E + C::EPB - 1) / C::EPB;
  constexpr bool PFG = !GLayout<P>::kTPE;   // slice-major factors: a group is one contiguous block
  auto group_bytes = [&](long long g) -> unsigned {
    long long nel = m.E - g * C::EPB;
    if (nel > C::EPB) nel = C::EPB;
    return (unsigned)(nel * 6 * N3 * sizeof(double));
  };
  if (PFG && threadIdx.x == 0 && blockIdx.x < ngroups)
    gauss_prefetch_l2(G + (long long)blockIdx.x * C::EPB * 6 * N3, group_bytes(blockIdx.x));
  for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const long long e = grp * C::EPB + le;
    const bool act = e < m.E;
    int ex = 0, ey = 0, ez = 0;
    if (act) elem_coords(m, e, ex, ey, ez);
    const long long nx = grp + gridDim.x;
    if (PFG && nx < ngroups) {   // next group: factors (thread 0) and this thread's u column
      if (threadIdx.x == 0) gauss_prefetch_l2(G + nx * C::EPB * 6 * N3, group_bytes(nx));
      const long long en = nx * C::EPB + le;
      if (en < m.E) {
        int qx, qy, qz;
        elem_coords(m, en, qx, qy, qz);
        const double* pu = u + (long long)(qx * P + t0) + (long long)m.Mx * (qy * P + t1) + sxy * (long long)(qz * P);
#pragma unroll
        for (int c = 0; c < N; ++c) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + sxy * c));
      }
    }
    __syncthreads();
    {  // gather: nodal column (a = t0, b = t1), masked (R4)
      const int I = ex * P + t0, J = ey * P + t1;
      const long long col = (long long)I + (long long)m.Mx * J + sxy * (long long)(ez * P);
#pragma unroll
      for (int c = 0; c < N; ++c) {
        const int K = ez * P + c;
        const bool bnd = DIR && (I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == 0 || K == m.Mz - 1);
        A[t0 + N * t1 + N2 * c] = (act && !bnd) ? __ldg(u + col + sxy * c) : 0.0;
      }
    }
    __syncthreads();
    {  // x-interpolation: line (b = t0, c = t1)
      double L[N], o[N];
#pragma unroll
      for (int a = 0; a < N; ++a) L[a] = A[a + N * t0 + N2 * t1];
      line_B<P, false>(L, o);
#pragma unroll
      for (int i = 0; i < N; ++i) Bb[i + N * t0 + N2 * t1] = o[i];
    }
    __syncthreads();
    {  // y-interpolation: line (i = t0, c = t1)
      double L[N], o[N];
#pragma unroll
      for (int b = 0; b < N; ++b) L[b] = Bb[t0 + N * b + N2 * t1];
      line_B<P, false>(L, o);
#pragma unroll
      for (int j = 0; j < N; ++j) A[t0 + N * j + N2 * t1] = o[j];
    }
    __syncthreads();
    double g2[N];
    {  // z-interpolation and z-gradient in registers: column (i = t0, j = t1)
      double L[N], uq[N];
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A[t0 + N * t1 + N2 * c];
      line_B<P, false>(L, uq);
      line_DG<P, false>(uq, g2);
#pragma unroll
      for (int k = 0; k < N; ++k) Cc[t0 + N * t1 + N2 * k] = uq[k];
    }
    __syncthreads();
    {  // x- and y-gradients on the Gauss grid: lines (j = t0, k = t1) -> A, (i = t0, k = t1) -> Bb
      double L[N], o[N], L2[N], o2[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) {
        L[mm] = Cc[mm + N * t0 + N2 * t1];
        L2[mm] = Cc[t0 + N * mm + N2 * t1];
      }
      line_DG<P, false>(L, o);
      line_DG<P, false>(L2, o2);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        A[i + N * t0 + N2 * t1] = o[i];
        Bb[t0 + N * i + N2 * t1] = o2[i];
      }
    }
    __syncthreads();
    double vz[N];
    {  // pointwise w = G g (G at the Gauss points), then D_G^T along z: column (i = t0, j = t1)
      double w2[N];
      const long long eg = act ? e : 0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int idx = t0 + N * t1 + N2 * k, ij = t0 + N * t1;
        const double G00 = __ldcs(G + GLayout<P>::off(eg, 0, ij, k)), G01 = __ldcs(G + GLayout<P>::off(eg, 1, ij, k));
        const double G02 = __ldcs(G + GLayout<P>::off(eg, 2, ij, k)), G11 = __ldcs(G + GLayout<P>::off(eg, 3, ij, k));
        const double G12 = __ldcs(G + GLayout<P>::off(eg, 4, ij, k)), G22 = __ldcs(G + GLayout<P>::off(eg, 5, ij, k));
        const double a0 = A[idx], a1 = Bb[idx], a2 = g2[k];
        A[idx] = G00 * a0 + G01 * a1 + G02 * a2;
        Bb[idx] = G01 * a0 + G11 * a1 + G12 * a2;
        w2[k] = G02 * a0 + G12 * a1 + G22 * a2;
      }
      line_DG<P, true>(w2, vz);
    }
    __syncthreads();
    {  // D_G^T on x-lines of A (in place) and y-lines of Bb (in place)
      double L[N], o[N], L2[N], o2[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) {
        L[mm] = A[mm + N * t0 + N2 * t1];
        L2[mm] = Bb[t0 + N * mm + N2 * t1];
      }
      line_DG<P, true>(L, o);
      line_DG<P, true>(L2, o2);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        A[i + N * t0 + N2 * t1] = o[i];
        Bb[t0 + N * i + N2 * t1] = o2[i];
      }
    }
    __syncthreads();
    {  // v_q, then B^T along z: column (i = t0, j = t1) -> Cc (nodal c)
      double vq[N], o[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int idx = t0 + N * t1 + N2 * k;
        vq[k] = A[idx] + Bb[idx] + vz[k];
      }
      line_B<P, true>(vq, o);
#pragma unroll
      for (int c = 0; c < N; ++c) Cc[t0 + N * t1 + N2 * c] = o[c];
    }
    __syncthreads();
    {  // B^T along y: line (i = t0, c = t1) -> A (nodal b)
      double L[N], o[N];
#pragma unroll
      for (int j = 0; j < N; ++j) L[j] = Cc[t0 + N * j + N2 * t1];
      line_B<P, true>(L, o);
#pragma unroll
      for (int b = 0; b < N; ++b) A[t0 + N * b + N2 * t1] = o[b];
    }
    __syncthreads();
    if (act) {  // B^T along x: line (b = t0, c = t1) -> nodal a, scatter (fp64 RED)
      double L[N], o[N];
#pragma unroll
      for (int i = 0; i < N; ++i) L[i] = A[i + N * t0 + N2 * t1];
      line_B<P, true>(L, o);
      const int J = ey * P + t0, K = ez * P + t1;
      const long long row = (long long)m.Mx * J + sxy * K + (long long)ex * P;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const int I = ex * P + a;
        const bool bnd = DIR && (I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == 0 || K == m.Mz - 1);
        if (!bnd) atomicAdd(v + row + a, o[a]);
      }
    }
  }
}

// ---------------------------------------------------------------------------- apply, v2 (3 <= p <= 16)
//
// The gradient at the Gauss points taken directly from the nodal values with DB = D_G B (ell_a'(xi_i)):
//   g0 = (DB x B x B) u, g1 = (B x DB x B) u, g2 = (B x B x DB) u,   v = the transposed chain of w = G g,
// sum-factorised as  x: Xb = B u, Xd = DB u;  y: Yb = B Xb, Yd = DB Xb, Y0 = B Xd;
// z (registers): g0 = B Y0, g1 = B Yd, g2 = DB Yb, w = G g, Z0 = B^T w0, Z1 = B^T w1, Z2 = DB^T w2;
// y^T: T0 = B^T Z0, Tb = DB^T Z1 + B^T Z2;  x^T: v = DB^T T0 + B^T Tb, RED.
// 16 line products instead of 12, but 5 block barriers per group instead of 11, three work arrays, every
// line read once per pass for all its products, and the even-odd split (even p) halves the FMAs.  The
// factors are staged like the collocated kernel's: one TMA bulk copy per group into shared memory,
// issued for group g+1 as soon as the z pass of group g has consumed the buffer, plus an L2 prefetch of
// group g+2 and of the next group's u columns; persistent blocks (grid = occupancy x SMs).

// out = M L on one line: SET 0 B, 1 DB, 2 B^T, 3 DB^T
template <int P, int SET>
__device__ __forceinline__ void gline(const double (&L)[P + 1], double (&out)[P + 1]) {
  constexpr int N = P + 1;
  if constexpr (P % 2 == 0 && P >= 4) {
    constexpr int c = P / 2, base = geoOffset(P) + SET * geoSize(P);
    constexpr bool sym = (SET == 0 || SET == 2);
    double ev[c], od[c];
#pragma unroll
    for (int m = 0; m < c; ++m) {
      ev[m] = L[m] + L[N - 1 - m];
      od[m] = L[m] - L[N - 1 - m];
    }
#pragma unroll
    for (int i = 0; i < c; ++i) {
      double T = c_gEO[base + 2 * c * c + i] * L[c], S = 0.0;
#pragma unroll
      for (int m = 0; m < c; ++m) {
        T = fma(c_gEO[base + i * c + m], ev[m], T);
        S = fma(c_gEO[base + c * c + i * c + m], od[m], S);
      }
      out[i] = T + S;
      out[N - 1 - i] = sym ? T - S : S - T;
    }
    double M = sym ? c_gEO[base + 2 * c * c + 2 * c] * L[c] : 0.0;
#pragma unroll
    for (int m = 0; m < c; ++m) M = fma(c_gEO[base + 2 * c * c + c + m], sym ? ev[m] : od[m], M);
    out[c] = M;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) {
        const double coef = SET == 0 ? c_qB[qOffset(P) + i * N + m]
                          : SET == 1 ? c_qDB[qOffset(P) + i * N + m]
                          : SET == 2 ? c_qB[qOffset(P) + m * N + i]
                                     : c_qDB[qOffset(P) + m * N + i];
        s = fma(coef, L[m], s);
      }
      out[i] = s;
    }
  }
}

// GS (p <= 8): the group's factors are staged in shared memory by TMA; p >= 9 (an element's factors are up
// to 236 KB): the pointwise pass reads them from L2 (streaming loads; the group was L2-prefetched).
template <int P>
struct GaussV2Cfg {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr bool GS = P <= 8;
  static constexpr int ARR = GS ? 9 : 3;           // n^3 arrays per element: (6 staged factors +) three work arrays
  static constexpr int PER_ELEM = ARR * N3 * 8;
  static constexpr int EPB_SMEM = 53000 / PER_ELEM > 0 ? 53000 / PER_ELEM : 1;
  static constexpr int EPB_THR = 256 / N2 > 0 ? 256 / N2 : 1;
  static constexpr int EPB = EPB_SMEM < EPB_THR ? EPB_SMEM : EPB_THR;
  static constexpr int THREADS = EPB * N2;
  static constexpr size_t SMEM = (size_t)EPB * PER_ELEM + 16;
  static constexpr int MINB_SMEM = (227 * 1024) / (SMEM + 1024) < 8 ? (227 * 1024) / (SMEM + 1024) : 8;
  static constexpr int MINB = GS ? MINB_SMEM : (P >= 12 ? 1 : 2);   // p >= 9: the register file decides
};

template <int P, bool DIR>
__global__ void __launch_bounds__(GaussV2Cfg<P>::THREADS, GaussV2Cfg<P>::MINB)
    k_apply_gauss_v2(MeshDev m, const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ v) {
  using C = GaussV2Cfg<P>;
  constexpr int N = C::N, N2 = C::N2, N3 = C::N3;
  constexpr bool GS = C::GS;
  extern __shared__ __align__(128) double gsm2[];
  double* sG = gsm2;                                   // [EPB][k][6][n^2] (GS)
  const int le = threadIdx.x / N2, t = threadIdx.x - le * N2, t0 = t % N, t1 = t / N;
  double* A0 = gsm2 + (GS ? C::EPB * 6 * N3 : 0) + le * 3 * N3;
  double* A1 = A0 + N3;
  double* A2 = A1 + N3;
  uint64_t* bar = (uint64_t*)(gsm2 + C::EPB * C::ARR * N3);
  const double* gE = sG + le * 6 * N3;
  const long long sxy = (long long)m.Mx * m.My;
  const long long ngroups = (m.E + C::EPB - 1) / C::EPB;
  const long long gstride = gridDim.x;
  auto group_bytes = [&](long long g) -> unsigned {
    long long nel = m.E - g * C::EPB;
    if (nel > C::EPB) nel = C::EPB;
    return (unsigned)(nel * 6 * N3 * sizeof(double));
  };
  auto prefetch_columns = [&](long long g) {
    const long long en = g * C::EPB + le;
    if (en >= m.E) return;
    int qx, qy, qz;
    elem_coords(m, en, qx, qy, qz);
    const double* pu = u + (long long)(qx * P + t0) + (long long)m.Mx * (qy * P + t1) + sxy * (long long)(qz * P);
#pragma unroll
    for (int c = 0; c < N; ++c) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + sxy * c));
  };
  long long grp = blockIdx.x;
  if (threadIdx.x == 0) {
    if (GS) {
      mbar_init(bar, 1);
      if (grp < ngroups) bulk_load(sG, G + grp * C::EPB * 6 * N3, group_bytes(grp), bar);
      if (grp + gstride < ngroups) gauss_prefetch_l2(G + (grp + gstride) * C::EPB * 6 * N3, group_bytes(grp + gstride));
    } else if (grp < ngroups) {
      gauss_prefetch_l2(G + grp * C::EPB * 6 * N3, group_bytes(grp));
    }
  }
  unsigned phase = 0;
  for (; grp < ngroups; grp += gstride) {
    const long long e = grp * C::EPB + le;
    const bool act = e < m.E;
    int ex = 0, ey = 0, ez = 0;
    if (act) elem_coords(m, e, ex, ey, ez);
    if (grp + gstride < ngroups) prefetch_columns(grp + gstride);
    {  // gather: nodal column (a = t0, b = t1), masked (R4)
      const int I = ex * P + t0, J = ey * P + t1;
      const long long col = (long long)I + (long long)m.Mx * J + sxy * (long long)(ez * P);
#pragma unroll
      for (int c = 0; c < N; ++c) {
        const int K = ez * P + c;
        const bool bnd = DIR && (I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == m.Kb0 || K == m.Kb1);
        A0[t + N2 * c] = (act && !bnd) ? __ldg(u + col + sxy * c) : 0.0;
      }
    }
    __syncthreads();
    {  // x: line (b = t0, c = t1): Xb = B u -> A1, Xd = DB u -> A2
      double L[N], o[N];
#pragma unroll
      for (int a = 0; a < N; ++a) L[a] = A0[a + N * t0 + N2 * t1];
      gline<P, 0>(L, o);
#pragma unroll
      for (int i = 0; i < N; ++i) A1[i + N * t0 + N2 * t1] = o[i];
      gline<P, 1>(L, o);
#pragma unroll
      for (int i = 0; i < N; ++i) A2[i + N * t0 + N2 * t1] = o[i];
    }
    __syncthreads();
    {  // y: line (i = t0, c = t1): Yb = B Xb -> A0, Yd = DB Xb -> A1 (in place), Y0 = B Xd -> A2 (in place)
      double L[N], o[N];
      const int yb = t0 + N2 * t1;
#pragma unroll
      for (int b = 0; b < N; ++b) L[b] = A1[yb + N * b];
      gline<P, 0>(L, o);
#pragma unroll
      for (int j = 0; j < N; ++j) A0[yb + N * j] = o[j];
      gline<P, 1>(L, o);
#pragma unroll
      for (int j = 0; j < N; ++j) A1[yb + N * j] = o[j];
#pragma unroll
      for (int b = 0; b < N; ++b) L[b] = A2[yb + N * b];
      gline<P, 0>(L, o);
#pragma unroll
      for (int j = 0; j < N; ++j) A2[yb + N * j] = o[j];
    }
    __syncthreads();
    if (GS) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    }
    if constexpr (GS) {  // z in registers: column (i = t0, j = t1)
      double L[N], g0[N], g1[N], g2[N];
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A2[t + N2 * c];
      gline<P, 0>(L, g0);
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A1[t + N2 * c];
      gline<P, 0>(L, g1);
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A0[t + N2 * c];
      gline<P, 1>(L, g2);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double G00, G01, G02, G11, G12, G22;
        if (GS) {
          const double* Gk = gE + gofs<N>(0, t, k);
          G00 = Gk[0]; G01 = Gk[N2]; G02 = Gk[2 * N2]; G11 = Gk[3 * N2]; G12 = Gk[4 * N2]; G22 = Gk[5 * N2];
        } else {
          const double* Gk = G + (act ? e : 0) * 6 * N3 + gofs<N>(0, t, k);
          G00 = __ldcs(Gk); G01 = __ldcs(Gk + N2); G02 = __ldcs(Gk + 2 * N2);
          G11 = __ldcs(Gk + 3 * N2); G12 = __ldcs(Gk + 4 * N2); G22 = __ldcs(Gk + 5 * N2);
        }
        const double a0 = g0[k], a1 = g1[k], a2 = g2[k];
        g0[k] = G00 * a0 + G01 * a1 + G02 * a2;
        g1[k] = G01 * a0 + G11 * a1 + G12 * a2;
        g2[k] = G02 * a0 + G12 * a1 + G22 * a2;
      }
      gline<P, 2>(g0, L);
#pragma unroll
      for (int c = 0; c < N; ++c) A2[t + N2 * c] = L[c];
      gline<P, 2>(g1, L);
#pragma unroll
      for (int c = 0; c < N; ++c) A1[t + N2 * c] = L[c];
      gline<P, 3>(g2, L);
#pragma unroll
      for (int c = 0; c < N; ++c) A0[t + N2 * c] = L[c];
    } else {  // p >= 9: the same z pass one line product at a time through the thread's own columns of
              // A0 / A1 / A2 (three 17-value register arrays at once would spill)
      double L[N], o[N];
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A2[t + N2 * c];
      gline<P, 0>(L, o);
#pragma unroll
      for (int k = 0; k < N; ++k) A2[t + N2 * k] = o[k];
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A1[t + N2 * c];
      gline<P, 0>(L, o);
#pragma unroll
      for (int k = 0; k < N; ++k) A1[t + N2 * k] = o[k];
#pragma unroll
      for (int c = 0; c < N; ++c) L[c] = A0[t + N2 * c];
      gline<P, 1>(L, o);   // g2 stays in registers (o)
      const double* Ge = G + (act ? e : 0) * 6 * N3;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double* Gk = Ge + gofs<N>(0, t, k);
        const double G00 = __ldcs(Gk), G01 = __ldcs(Gk + N2), G02 = __ldcs(Gk + 2 * N2);
        const double G11 = __ldcs(Gk + 3 * N2), G12 = __ldcs(Gk + 4 * N2), G22 = __ldcs(Gk + 5 * N2);
        const double a0 = A2[t + N2 * k], a1 = A1[t + N2 * k], a2 = o[k];
        A2[t + N2 * k] = G00 * a0 + G01 * a1 + G02 * a2;
        A1[t + N2 * k] = G01 * a0 + G11 * a1 + G12 * a2;
        o[k] = G02 * a0 + G12 * a1 + G22 * a2;
      }
      gline<P, 3>(o, L);
#pragma unroll
      for (int c = 0; c < N; ++c) A0[t + N2 * c] = L[c];
#pragma unroll
      for (int k = 0; k < N; ++k) L[k] = A2[t + N2 * k];
      gline<P, 2>(L, o);
#pragma unroll
      for (int c = 0; c < N; ++c) A2[t + N2 * c] = o[c];
#pragma unroll
      for (int k = 0; k < N; ++k) L[k] = A1[t + N2 * k];
      gline<P, 2>(L, o);
#pragma unroll
      for (int c = 0; c < N; ++c) A1[t + N2 * c] = o[c];
    }
    __syncthreads();
    {  // factors consumed: next group's TMA copy and the L2 prefetch of the group after
      const long long nx = grp + gstride;
      if (nx < ngroups && threadIdx.x == 0) {
        if (GS) {
          fence_proxy_async_smem();
          bulk_load(sG, G + nx * C::EPB * 6 * N3, group_bytes(nx), bar);
          if (nx + gstride < ngroups) gauss_prefetch_l2(G + (nx + gstride) * C::EPB * 6 * N3, group_bytes(nx + gstride));
        } else {
          gauss_prefetch_l2(G + nx * C::EPB * 6 * N3, group_bytes(nx));
        }
      }
    }
    {  // y^T: line (i = t0, c = t1): T0 = B^T Z0 -> A2 (in place), Tb = DB^T Z1 + B^T Z2 -> A1 (in place)
      double L[N], o[N], o2[N];
      const int yb = t0 + N2 * t1;
#pragma unroll
      for (int j = 0; j < N; ++j) L[j] = A2[yb + N * j];
      gline<P, 2>(L, o);
#pragma unroll
      for (int b = 0; b < N; ++b) A2[yb + N * b] = o[b];
#pragma unroll
      for (int j = 0; j < N; ++j) L[j] = A1[yb + N * j];
      gline<P, 3>(L, o);
#pragma unroll
      for (int j = 0; j < N; ++j) L[j] = A0[yb + N * j];
      gline<P, 2>(L, o2);
#pragma unroll
      for (int b = 0; b < N; ++b) A1[yb + N * b] = o[b] + o2[b];
    }
    __syncthreads();
    if (act) {  // x^T: line (b = t0, c = t1): v = DB^T T0 + B^T Tb, scatter (fp64 RED)
      double L[N], o[N], o2[N];
#pragma unroll
      for (int i = 0; i < N; ++i) L[i] = A2[i + N * t0 + N2 * t1];
      gline<P, 3>(L, o);
#pragma unroll
      for (int i = 0; i < N; ++i) L[i] = A1[i + N * t0 + N2 * t1];
      gline<P, 2>(L, o2);
      const int J = ey * P + t0, K = ez * P + t1;
      const long long row = (long long)m.Mx * J + sxy * K + (long long)ex * P;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const int I = ex * P + a;
        const bool bnd = DIR && (I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == m.Kb0 || K == m.Kb1);
        if (!bnd) atomicAdd(v + row + a, o[a] + o2[a]);
      }
    }
    // (the next gather writes A0, last read before the barrier above; A1 / A2 are rewritten only after
    //  the barrier that follows the gather)
  }
}

// ---------------------------------------------------------------------------- diagonal

// d_l = sum_q grad phi_l(q)^T G_q grad phi_l(q), grad phi_l(q) = (DB_ia B_jb B_kc, B_ia DB_jb B_kc,
// B_ia B_jb DB_kc): block per element, thread per node, n^3 points each (setup only).
template <int P>
__global__ void __launch_bounds__(256) k_diag_gauss(MeshDev m, int bc, const double* __restrict__ G, double* d) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  __shared__ double sB[N2], sDB[N2];
  for (int t = threadIdx.x; t < N2; t += blockDim.x) {
    sB[t] = c_qB[qOffset(P) + t];
    sDB[t] = c_qDB[qOffset(P) + t];
  }
  __syncthreads();
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    for (int l = threadIdx.x; l < N3; l += blockDim.x) {
      const int a = l % N, b = (l / N) % N, c = l / N2;
      const long long g = (long long)(ex * P + a) + (long long)m.Mx * ((long long)(ey * P + b) + (long long)m.My * (ez * P + c));
      if (bc == 0 && lattice_boundary(m, g)) continue;
      double s = 0.0;
      for (int k = 0; k < N; ++k) {
        const double Bk = sB[k * N + c], Dk = sDB[k * N + c];
        for (int j = 0; j < N; ++j) {
          const double Bj = sB[j * N + b], Dj = sDB[j * N + b];
          for (int i = 0; i < N; ++i) {
            const double Bi = sB[i * N + a], Di = sDB[i * N + a];
            const double d0 = Di * Bj * Bk, d1 = Bi * Dj * Bk, d2 = Bi * Bj * Dk;
            const int ij = i + N * j;
            const double G00 = G[GLayout<P>::off(e, 0, ij, k)], G01 = G[GLayout<P>::off(e, 1, ij, k)];
            const double G02 = G[GLayout<P>::off(e, 2, ij, k)], G11 = G[GLayout<P>::off(e, 3, ij, k)];
            const double G12 = G[GLayout<P>::off(e, 4, ij, k)], G22 = G[GLayout<P>::off(e, 5, ij, k)];
            s += d0 * (G00 * d0 + 2.0 * (G01 * d1 + G02 * d2)) + d1 * (G11 * d1 + 2.0 * G12 * d2) + d2 * G22 * d2;
          }
        }
      }
      atomicAdd(d + g, s);
    }
  }
}

// ---------------------------------------------------------------------------- load vector

// Manufactured load (rhs 1): b_l = sum_q phi_l(x_q) wG_q detJ_q f(x_q), f = -div(mu grad u*) with
// u* = sin(pi x) sin(pi y) sin(pi z); interior rows only.  Block per element: F_q in smem, then
// the B^T x B^T x B^T contraction per node (setup only).
template <int P>
__global__ void __launch_bounds__(256) k_load_gauss(MeshDev m, double* f) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  extern __shared__ double lsm[];
  double* X = lsm;            // [3][N3]
  double* F = X + 3 * N3;     // [N3]
  double* sB = F + N3;        // [N2]
  double* sDB = sB + N2;      // [N2]
  const double* w = c_qw + qvOffset(P);
  const double pi = 3.141592653589793238463;
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    __syncthreads();
    load_tables_and_nodes<P>(m, e, X, sB, sDB);
    __syncthreads();
    for (int q = threadIdx.x; q < N3; q += blockDim.x) {
      const int i = q % N, j = (q / N) % N, k = q / N2;
      double J[3][3], xq[3];
      gauss_jacobian<P>(X, sB, sDB, i, j, k, J, xq);
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      const double x = xq[0], y = xq[1], z = xq[2];
      const double sx = sinpi(x), sy = sinpi(y), sz = sinpi(z);
      const double us = sx * sy * sz;
      const double gu[3] = {pi * cospi(x) * sy * sz, pi * sx * cospi(y) * sz, pi * sx * sy * cospi(z)};
      const double mu = coeff_mu(m, x, y, z);
      double gm[3];
      coeff_grad(m, x, y, z, mu, gm);
      const double fx = 3.0 * pi * pi * mu * us - (gm[0] * gu[0] + gm[1] * gu[1] + gm[2] * gu[2]);
      F[q] = w[i] * w[j] * w[k] * det * fx;
    }
    __syncthreads();
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    for (int l = threadIdx.x; l < N3; l += blockDim.x) {
      const int a = l % N, b = (l / N) % N, c = l / N2;
      const long long g = (long long)(ex * P + a) + (long long)m.Mx * ((long long)(ey * P + b) + (long long)m.My * (ez * P + c));
      if (lattice_boundary(m, g)) continue;
      double s = 0.0;
      for (int k = 0; k < N; ++k)
        for (int j = 0; j < N; ++j) {
          const double bjk = sB[j * N + b] * sB[k * N + c];
          for (int i = 0; i < N; ++i) s += sB[i * N + a] * bjk * F[i + N * (j + N * k)];
        }
      atomicAdd(f + g, s);
    }
  }
}

// ---------------------------------------------------------------------------- coarse CG

// Single-CTA CG on a small Gauss level (the coarsest p = 1 / 2 levels of a Gauss hierarchy; R13):
// vectors in global memory (L2-resident), thread-per-element inline apply with the Gauss tables.
template <int P>
__device__ void cta_apply_gauss(const MeshDev& m, const double* __restrict__ G, const double* x, double* y) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  for (long long g = threadIdx.x; g < m.N; g += blockDim.x) y[g] = lattice_boundary(m, g) ? __ldcg(x + g) : 0.0;
  __syncthreads();
  for (long long e = threadIdx.x; e < m.E; e += blockDim.x) {
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    double ue[N3], t1[N3], t2[N3];
    long long gl[N3];
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          const int l = a + N * (b + N * c);
          const long long g = (long long)(ex * P + a) + (long long)m.Mx * ((long long)(ey * P + b) + (long long)m.My * (ez * P + c));
          const bool bnd = lattice_boundary(m, g);
          gl[l] = bnd ? -1 : g;
          ue[l] = bnd ? 0.0 : __ldcg(x + g);
        }
    // u_q = (B x B x B) u_e
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < N; ++a) s = fma(qB<P>(i, a), ue[a + N * (b + N * c)], s);
          t1[i + N * (b + N * c)] = s;
        }
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < N; ++b) s = fma(qB<P>(j, b), t1[i + N * (b + N * c)], s);
          t2[i + N * (j + N * c)] = s;
        }
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < N; ++c) s = fma(qB<P>(k, c), t2[i + N * (j + N * c)], s);
          ue[i + N * (j + N * k)] = s;   // u_q
          t1[i + N * (j + N * k)] = 0.0;  // v_q accumulator
        }
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double g0 = 0, g1 = 0, g2 = 0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) {
            g0 = fma(qDG<P>(i, mm), ue[mm + N * (j + N * k)], g0);
            g1 = fma(qDG<P>(j, mm), ue[i + N * (mm + N * k)], g1);
            g2 = fma(qDG<P>(k, mm), ue[i + N * (j + N * mm)], g2);
          }
          const int ij = i + N * j;
          const double G00 = G[GLayout<P>::off(e, 0, ij, k)], G01 = G[GLayout<P>::off(e, 1, ij, k)];
          const double G02 = G[GLayout<P>::off(e, 2, ij, k)], G11 = G[GLayout<P>::off(e, 3, ij, k)];
          const double G12 = G[GLayout<P>::off(e, 4, ij, k)], G22 = G[GLayout<P>::off(e, 5, ij, k)];
          const double w0 = G00 * g0 + G01 * g1 + G02 * g2;
          const double w1 = G01 * g0 + G11 * g1 + G12 * g2;
          const double w2 = G02 * g0 + G12 * g1 + G22 * g2;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) {
            t1[mm + N * (j + N * k)] = fma(qDG<P>(i, mm), w0, t1[mm + N * (j + N * k)]);
            t1[i + N * (mm + N * k)] = fma(qDG<P>(j, mm), w1, t1[i + N * (mm + N * k)]);
            t1[i + N * (j + N * mm)] = fma(qDG<P>(k, mm), w2, t1[i + N * (j + N * mm)]);
          }
        }
    // v_e = (B^T x B^T x B^T) v_q
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) s = fma(qB<P>(i, a), t1[i + N * (j + N * k)], s);
          t2[a + N * (j + N * k)] = s;
        }
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) s = fma(qB<P>(j, b), t2[a + N * (j + N * k)], s);
          t1[a + N * (b + N * k)] = s;
        }
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s = fma(qB<P>(k, c), t1[a + N * (b + N * k)], s);
          const int l = a + N * (b + N * c);
          if (gl[l] >= 0) atomicAdd(y + gl[l], s);
        }
  }
  __threadfence_block();
  __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(256) k_coarse_cg_gauss(MeshDev m, const double* __restrict__ G, const double* b,
                                                          double* x, double* r, double* p, double* q, double* scal,
                                                          double rtol, int maxit) {
  __shared__ double red[32];
  const long long n = m.N;
  double rr = 0.0;
  for (long long g = threadIdx.x; g < n; g += blockDim.x) {
    const double bg = b[g];
    x[g] = 0.0; r[g] = bg; p[g] = bg;
    rr += bg * bg;
  }
  rr = block_sum(rr, red);
  const double bn = sqrt(rr);
  int it = 0, status = 0;
  if (bn > 0.0) {
    for (; it < maxit; ++it) {
      if (sqrt(rr) <= rtol * bn) break;
      __syncthreads();
      cta_apply_gauss<P>(m, G, p, q);
      double pq = 0.0;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) pq += __ldcg(p + g) * __ldcg(q + g);
      pq = block_sum(pq, red);
      if (!(pq > 0.0)) { status = 6; break; }
      const double alpha = rr / pq;
      double rn = 0.0;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) {
        x[g] = __ldcg(x + g) + alpha * __ldcg(p + g);
        const double rg = __ldcg(r + g) - alpha * __ldcg(q + g);
        r[g] = rg;
        rn += rg * rg;
      }
      rn = block_sum(rn, red);
      const double beta = rn / rr;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) p[g] = __ldcg(r + g) + beta * __ldcg(p + g);
      rr = rn;
      __threadfence_block();
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) { scal[8] = (double)it; scal[9] = sqrt(rr); scal[10] = (double)status; }
}

// ---------------------------------------------------------------------------- launchers

#define SFMG_GAUSS_DISPATCH(p, F, ...)  \
  switch (p) {                          \
    case 1: return F<1>(__VA_ARGS__);   \
    case 2: return F<2>(__VA_ARGS__);   \
    case 3: return F<3>(__VA_ARGS__);   \
    case 4: return F<4>(__VA_ARGS__);   \
    case 5: return F<5>(__VA_ARGS__);   \
    case 6: return F<6>(__VA_ARGS__);   \
    case 7: return F<7>(__VA_ARGS__);   \
    case 8: return F<8>(__VA_ARGS__);   \
    case 9: return F<9>(__VA_ARGS__);   \
    case 10: return F<10>(__VA_ARGS__); \
    case 11: return F<11>(__VA_ARGS__); \
    case 12: return F<12>(__VA_ARGS__); \
    case 13: return F<13>(__VA_ARGS__); \
    case 14: return F<14>(__VA_ARGS__); \
    case 15: return F<15>(__VA_ARGS__); \
    case 16: return F<16>(__VA_ARGS__); \
  }                                     \
  return cudaErrorInvalidValue;

static unsigned elem_grid(long long E) { return (unsigned)(E < 148LL * 8 ? (E > 0 ? E : 1) : 148LL * 8); }

template <int P>
static cudaError_t geometry_g(const MeshDev& m, double* G, int* bad, cudaStream_t s) {
  constexpr int N = P + 1;
  const size_t smem = sizeof(double) * (3 * N * N * N + 2 * N * N);
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_geometry_gauss<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  k_geometry_gauss<P><<<elem_grid(m.E), 256, smem, s>>>(m, G, bad);
  return cudaGetLastError();
}
cudaError_t launch_geometry_gauss(const MeshDev& m, double* G, int* bad, cudaStream_t s) {
  cudaError_t e = upload_gauss_tables(m.p);
  if (e) return e;
  SFMG_GAUSS_DISPATCH(m.p, geometry_g, m, G, bad, s);
}

// SFMG_GAUSS_V1=1: the round-1 kernel for every order (A/B measurements)
static bool gauss_v1_forced() {
  static const bool on = [] {
    const char* e = getenv("SFMG_GAUSS_V1");
    return e && e[0] == '1';
  }();
  return on;
}

template <int P, bool DIR>
static cudaError_t apply_g_v2(const MeshDev& m, const double* G, const double* u, double* v, cudaStream_t s) {
  using C = GaussV2Cfg<P>;
  static IntPerDevice occ;
  int per_sm = 0;
  cudaError_t e = occ.get(per_sm, [&](int& n) {
    cudaError_t r = cudaFuncSetAttribute(k_apply_gauss_v2<P, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (r) return r;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_apply_gauss_v2<P, DIR>, C::THREADS, C::SMEM);
  });
  if (e) return e;
  const long long groups = (m.E + C::EPB - 1) / C::EPB;
  long long grid = (long long)per_sm * num_sms();
  if (grid > groups) grid = groups;
  k_apply_gauss_v2<P, DIR><<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(m, G, u, v);
  return cudaGetLastError();
}

template <int P>
static cudaError_t apply_g(const MeshDev& m, int bc, const double* G, const double* u, double* v, cudaStream_t s) {
  if constexpr (P >= 3 && P <= kGaussV2MaxP) {
    if (!gauss_v1_forced())
      return bc == 0 ? apply_g_v2<P, true>(m, G, u, v, s) : apply_g_v2<P, false>(m, G, u, v, s);
  }
  using C = GaussCfg<P>;
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_apply_gauss<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
      if (e) return e;
      e = cudaFuncSetAttribute(k_apply_gauss<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  const long long groups = (m.E + C::EPB - 1) / C::EPB;
  const unsigned grid = (unsigned)(groups < 148LL * 16 ? groups : 148LL * 16);
  if (bc == 0) k_apply_gauss<P, true><<<grid, C::THREADS, C::SMEM, s>>>(m, G, u, v);
  else k_apply_gauss<P, false><<<grid, C::THREADS, C::SMEM, s>>>(m, G, u, v);
  return cudaGetLastError();
}
cudaError_t launch_apply_gauss(const MeshDev& m, int bc, const double* G, const double* u, double* v, cudaStream_t s) {
  SFMG_GAUSS_DISPATCH(m.p, apply_g, m, bc, G, u, v, s);
}

template <int P>
static cudaError_t diag_g(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s) {
  k_diag_gauss<P><<<elem_grid(m.E), 256, 0, s>>>(m, bc, G, d);
  return cudaGetLastError();
}
cudaError_t launch_diag_gauss(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s) {
  SFMG_GAUSS_DISPATCH(m.p, diag_g, m, bc, G, d, s);
}

template <int P>
static cudaError_t load_g(const MeshDev& m, double* f, cudaStream_t s) {
  constexpr int N = P + 1;
  const size_t smem = sizeof(double) * (4 * N * N * N + 2 * N * N);
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_load_gauss<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  k_load_gauss<P><<<elem_grid(m.E), 256, smem, s>>>(m, f);
  return cudaGetLastError();
}
cudaError_t launch_load_gauss(const MeshDev& m, double* f, cudaStream_t s) {
  cudaError_t e = upload_gauss_tables(m.p);
  if (e) return e;
  SFMG_GAUSS_DISPATCH(m.p, load_g, m, f, s);
}

cudaError_t launch_coarse_cg_gauss(const MeshDev& m, const double* G, const double* b, double* x, double* r,
                                   double* p, double* q, double* scal, double rtol, int maxit, cudaStream_t s) {
  if (m.p == 1) k_coarse_cg_gauss<1><<<1, 256, 0, s>>>(m, G, b, x, r, p, q, scal, rtol, maxit);
  else if (m.p == 2) k_coarse_cg_gauss<2><<<1, 256, 0, s>>>(m, G, b, x, r, p, q, scal, rtol, maxit);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace sfmg

// Host construction of the 1-D LGL tables (eq. (7)
// P:400-408).  Small fp64 arrays (n <= 17) that are uploaded once per order to __constant__.
//
// Nodes: the Lobatto iteration x <- x - (x P_p - P_{p-1}) / ((p+1) P_p), whose fixed points are
// the zeros of (1 - x^2) P_p'(x), started from Chebyshev-Gauss-Lobatto points, then sorted and
// symmetrised (exact 0 at the centre for even p).  Weights 2 / (p (p+1) P_p(x_i)^2).
// Derivative and interpolation matrices use the barycentric form of Lagrange interpolation.
#include <algorithm>
#include <cmath>

#include "sfmg_internal.h"

namespace sfmg {

static void legendre_pair(int p, double x, double* Pp, double* Pm1) {
  double a = 1.0, b = x;   // P_0, P_1
  if (p == 0) { *Pp = 1.0; *Pm1 = 0.0; return; }
  for (int k = 2; k <= p; ++k) {
    double c = ((2 * k - 1) * x * b - (k - 1) * a) / k;
    a = b; b = c;
  }
  *Pp = b; *Pm1 = a;
}

Basis1D make_basis(int p) {
  Basis1D B;
  B.p = p; B.n = p + 1;
  const int n = B.n;
  const double pi = 3.14159265358979323846;
  B.x.resize(n);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(pi * i / p);
    for (int it = 0; it < 100; ++it) {
      double Pp, Pm1;
      legendre_pair(p, x, &Pp, &Pm1);
      double dx = (x * Pp - Pm1) / ((p + 1) * Pp);
      x -= dx;
      if (std::fabs(dx) <= 1e-16) break;
    }
    B.x[i] = x;
  }
  std::sort(B.x.begin(), B.x.end());
  B.x[0] = -1.0; B.x[p] = 1.0;
  for (int i = 1; i < n / 2; ++i) {
    double h = 0.5 * (B.x[p - i] - B.x[i]);
    B.x[i] = -h; B.x[p - i] = h;
  }
  if (p % 2 == 0) B.x[p / 2] = 0.0;
  B.w.resize(n);
  for (int i = 0; i < n; ++i) {
    double Pp, Pm1;
    legendre_pair(p, B.x[i], &Pp, &Pm1);
    B.w[i] = 2.0 / (p * (p + 1.0) * Pp * Pp);
  }
  // barycentric weights and D_ij = (lam_j / lam_i) / (x_i - x_j), D_ii = -sum_{j != i} D_ij
  std::vector<double> lam(n, 1.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) lam[j] /= (B.x[j] - B.x[k]);
  B.D.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      double d = (lam[j] / lam[i]) / (B.x[i] - B.x[j]);
      B.D[i * n + j] = d;
      s += d;
    }
    B.D[i * n + i] = -s;
  }
  return B;
}

std::vector<double> make_interp(int pc, int pf) {
  Basis1D C = make_basis(pc), F = make_basis(pf);
  const int nc = C.n, nf = F.n;
  std::vector<double> lam(nc, 1.0);
  for (int j = 0; j < nc; ++j)
    for (int k = 0; k < nc; ++k)
      if (k != j) lam[j] /= (C.x[j] - C.x[k]);
  std::vector<double> I(nf * nc, 0.0);
  for (int i = 0; i < nf; ++i) {
    const double t = F.x[i];
    int hit = -1;
    for (int a = 0; a < nc; ++a)
      if (t == C.x[a]) hit = a;
    if (hit >= 0) { I[i * nc + hit] = 1.0; continue; }
    double den = 0.0;
    for (int a = 0; a < nc; ++a) den += lam[a] / (t - C.x[a]);
    for (int a = 0; a < nc; ++a) I[i * nc + a] = (lam[a] / (t - C.x[a])) / den;
  }
  return I;
}

// h-transfer at one order (NEXT-4; eq. (7) across nested meshes, R25): child s (0 = lower, 1 =
// upper half) of a coarse element; H[i*n + a] = ell_a(xi_i), xi_i = (xhat_i + 2 s - 1) / 2 the
// coarse-element coordinate of the child's node i.
std::vector<double> make_h_interp(int p, int s) {
  Basis1D B = make_basis(p);
  const int n = B.n;
  std::vector<double> lam(n, 1.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) lam[j] /= (B.x[j] - B.x[k]);
  std::vector<double> H(n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    const double t = 0.5 * (B.x[i] + 2.0 * s - 1.0);
    int hit = -1;
    for (int a = 0; a < n; ++a)
      if (t == B.x[a]) hit = a;
    if (hit >= 0) { H[i * n + hit] = 1.0; continue; }
    double den = 0.0;
    for (int a = 0; a < n; ++a) den += lam[a] / (t - B.x[a]);
    for (int a = 0; a < n; ++a) H[i * n + a] = (lam[a] / (t - B.x[a])) / den;
  }
  return H;
}

}  // namespace sfmg

// 2-D quadrilateral variant of the operator kernels (the paper's 2-D problems,
// P:875-890, discretised as in 3-D): order-p tensor LGL nodal basis on quadrilaterals,
// isoparametric geometry, collocated LGL (R1) or Gauss-Legendre (NEXT-3) quadrature.  A 2-D level is a
// lattice of Mx x My nodes (Mz = 1, no z boundary planes: MeshDev::Kb0 = Kb1 = -1), so the vector
// kernels (init, Chebyshev update, power iteration, reductions) are shared with 3-D.
//
// Element operator with 1-D tables at the quadrature points, B[i][a] = ell_a(q_i), DB[i][a] = ell_a'(q_i):
//   g0(i,j) = sum_ab DB[i][a] B[j][b] u(a,b),  g1(i,j) = sum_ab B[i][a] DB[j][b] u(a,b)
//   (w0, w1) = G_q (g0, g1),  G_q = w_i w_j mu(x_q) detJ_q J_q^{-1} J_q^{-T}  (3 unique values)
//   v(a,b) = sum_ij DB[i][a] B[j][b] w0(i,j) + B[i][a] DB[j][b] w1(i,j)
// evaluated sum-factorised in shared memory, one block per element; collocated LGL has B = I and
// skips those contractions.
#include <cmath>

#include "k_common.cuh"

namespace sfmg {

constexpr int q2Offset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += (q + 1) * (q + 1);
  return s;
}
constexpr int q2vOffset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += q + 1;
  return s;
}
__constant__ double c2_DB[2][q2Offset(kMaxOrder + 1)];   // [quad]: LGL D / Gauss DB
__constant__ double c2_B[q2Offset(kMaxOrder + 1)];       // Gauss B (LGL: identity)
__constant__ double c2_w[2][q2vOffset(kMaxOrder + 1)];   // [quad] quadrature weights
__constant__ double c2_x[q2vOffset(kMaxOrder + 1)];      // LGL nodes
static OncePerDevice g_2d_uploaded[2][kMaxOrder + 1];

cudaError_t upload_2d_tables(int p, int quad) {
  if (p < 1 || p > kMaxOrder || (quad != 0 && quad != 1)) return cudaErrorInvalidValue;
  return g_2d_uploaded[quad][p].run([&]() -> cudaError_t {
  const int n = p + 1;
  std::vector<double> xn, B, DB, w;
  quad_tables_1d(p, quad, xn, B, DB, w);
  const size_t mo = sizeof(double) * q2Offset(p), vo = sizeof(double) * q2vOffset(p);
  const size_t mq = sizeof(double) * q2Offset(kMaxOrder + 1), vq = sizeof(double) * q2vOffset(kMaxOrder + 1);
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(c2_DB, DB.data(), sizeof(double) * n * n, quad * mq + mo))) return e;
  if (quad == 1 && (e = cudaMemcpyToSymbol(c2_B, B.data(), sizeof(double) * n * n, mo))) return e;
  if ((e = cudaMemcpyToSymbol(c2_w, w.data(), sizeof(double) * n, quad * vq + vo))) return e;
  if ((e = cudaMemcpyToSymbol(c2_x, xn.data(), sizeof(double) * n, vo))) return e;
  return cudaSuccess;
  });
}

// tables of order P, quadrature Q into shared memory (B = I for collocated LGL)
template <int P, int Q>
__device__ __forceinline__ void load_tables2(double* sB, double* sDB, double* sw, double* sx) {
  constexpr int N = P + 1;
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) {
    sDB[t] = c2_DB[Q][q2Offset(P) + t];
    sB[t] = Q ? c2_B[q2Offset(P) + t] : ((t / N == t % N) ? 1.0 : 0.0);
  }
  for (int t = threadIdx.x; t < N; t += blockDim.x) {
    sw[t] = c2_w[Q][q2vOffset(P) + t];
    sx[t] = c2_x[q2vOffset(P) + t];
  }
}

// mu in 2-D (R6): 0 c0 (2d-const); 1 exp(c1 S), 2 10^(c1 S), S = sin 2pi x sin 2pi y; 3 c0 + c1 (cos^2 2pi x +
// cos^2 2pi y) (2d-var); 4 c0 + c1 (cos^2 10pi x + cos^2 10pi y) (2d-var')
__device__ __forceinline__ double mu2(const MeshDev& m, double x, double y) {
  switch (m.coeff) {
    case 0: return m.c0;
    case 1: return exp(m.c1 * sinpi(2.0 * x) * sinpi(2.0 * y));
    case 2: return exp10(m.c1 * sinpi(2.0 * x) * sinpi(2.0 * y));
    case 3: { const double a = cospi(2.0 * x), b = cospi(2.0 * y); return m.c0 + m.c1 * (a * a + b * b); }
    case 4: { const double a = cospi(10.0 * x), b = cospi(10.0 * y); return m.c0 + m.c1 * (a * a + b * b); }
  }
  return 0.0;
}
__device__ __forceinline__ void mu2_grad(const MeshDev& m, double x, double y, double mu, double g[2]) {
  const double tp = 6.283185307179586476925;
  const double dS0 = tp * cospi(2.0 * x) * sinpi(2.0 * y), dS1 = tp * sinpi(2.0 * x) * cospi(2.0 * y);
  switch (m.coeff) {
    case 1: g[0] = m.c1 * mu * dS0; g[1] = m.c1 * mu * dS1; return;
    case 2: g[0] = 2.302585092994045684 * m.c1 * mu * dS0; g[1] = 2.302585092994045684 * m.c1 * mu * dS1; return;
    case 3: g[0] = -tp * m.c1 * sinpi(4.0 * x); g[1] = -tp * m.c1 * sinpi(4.0 * y); return;   // d/dx cos^2(2 pi x)
    case 4: g[0] = -5.0 * tp * m.c1 * sinpi(20.0 * x); g[1] = -5.0 * tp * m.c1 * sinpi(20.0 * y); return;
  }
  g[0] = g[1] = 0.0;
}

// element nodes (reference square + the 2-D warp x_i += a sin pi X sin pi Y, R5) into sX[2][n^2]
template <int P>
__device__ __forceinline__ void nodes2(const MeshDev& m, const double* sx, int ex, int ey, double* sX) {
  constexpr int N = P + 1, N2 = N * N;
  for (int l = threadIdx.x; l < N2; l += blockDim.x) {
    const int a = l % N, b = l / N;
    const double Xr = (ex + 0.5 * (sx[a] + 1.0)) / m.nex, Yr = (ey + 0.5 * (sx[b] + 1.0)) / m.ney;
    const double s = (m.warp == 1) ? m.amp * sinpi(Xr) * sinpi(Yr) : 0.0;
    sX[l] = Xr + s;
    sX[N2 + l] = Yr + s;
  }
}

// J = d x / d xi and x at quadrature point (i, j) from the nodal positions (isoparametric, R2)
template <int P>
__device__ __forceinline__ void jac2(const double* sX, const double* sB, const double* sDB, int i, int j,
                                     double J[2][2], double xq[2]) {
  constexpr int N = P + 1, N2 = N * N;
  J[0][0] = J[0][1] = J[1][0] = J[1][1] = xq[0] = xq[1] = 0.0;
  for (int b = 0; b < N; ++b) {
    const double Bj = sB[j * N + b], Dj = sDB[j * N + b];
    for (int a = 0; a < N; ++a) {
      const double Bi = sB[i * N + a], Di = sDB[i * N + a];
      const double X = sX[a + N * b], Y = sX[N2 + a + N * b];
      J[0][0] += X * Di * Bj; J[0][1] += X * Bi * Dj;
      J[1][0] += Y * Di * Bj; J[1][1] += Y * Bi * Dj;
      xq[0] += X * Bi * Bj; xq[1] += Y * Bi * Bj;
    }
  }
}

__device__ __forceinline__ bool bnd2(const MeshDev& m, int I, int J) {
  return I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1;
}

template <int P, int Q>
__global__ void __launch_bounds__(128) k_geometry2d(MeshDev m, double* __restrict__ G, int* bad) {
  constexpr int N = P + 1, N2 = N * N;
  __shared__ double sB[N2], sDB[N2], sw[N], sx[N], sX[2 * N2];
  load_tables2<P, Q>(sB, sDB, sw, sx);
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    const int ex = (int)(e % m.nex), ey = (int)(e / m.nex);
    __syncthreads();
    nodes2<P>(m, sx, ex, ey, sX);
    __syncthreads();
    for (int q = threadIdx.x; q < N2; q += blockDim.x) {
      const int i = q % N, j = q / N;
      double J[2][2], xq[2];
      jac2<P>(sX, sB, sDB, i, j, J, xq);
      const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      if (!(det > 0.0)) atomicAdd(bad, 1);
      const double id = 1.0 / det;
      const double a00 = J[1][1] * id, a01 = -J[0][1] * id, a10 = -J[1][0] * id, a11 = J[0][0] * id;   // J^{-1}
      const double s = sw[i] * sw[j] * mu2(m, xq[0], xq[1]) * det;
      double* Ge = G + e * 3 * N2;
      Ge[q] = s * (a00 * a00 + a01 * a01);
      Ge[N2 + q] = s * (a00 * a10 + a01 * a11);
      Ge[2 * N2 + q] = s * (a10 * a10 + a11 * a11);
    }
  }
}

// v += A (M u) on interior nodes (DIR) / all nodes; v initialised by the caller (launch_init)
template <int P, int Q, bool DIR>
__global__ void __launch_bounds__(128) k_apply2d(MeshDev m, const double* __restrict__ G, const double* __restrict__ u,
                                                 double* __restrict__ v) {
  constexpr int N = P + 1, N2 = N * N;
  __shared__ double sB[N2], sDB[N2], sw[N], sx[N];
  __shared__ double su[N2], s0[N2], s1[N2], t0[Q ? N2 : 1], t1[Q ? N2 : 1];
  load_tables2<P, Q>(sB, sDB, sw, sx);
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    const int ex = (int)(e % m.nex), ey = (int)(e / m.nex);
    const double* Ge = G + e * 3 * N2;
    __syncthreads();
    for (int l = threadIdx.x; l < N2; l += blockDim.x) {
      const int a = l % N, b = l / N, I = ex * P + a, J = ey * P + b;
      su[l] = (DIR && bnd2(m, I, J)) ? 0.0 : u[I + (long long)m.Mx * J];
    }
    __syncthreads();
    if constexpr (Q == 0) {
      for (int q = threadIdx.x; q < N2; q += blockDim.x) {
        const int i = q % N, j = q / N;
        double g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          g0 += sDB[i * N + k] * su[k + N * j];
          g1 += sDB[j * N + k] * su[i + N * k];
        }
        s0[q] = Ge[q] * g0 + Ge[N2 + q] * g1;
        s1[q] = Ge[N2 + q] * g0 + Ge[2 * N2 + q] * g1;
      }
      __syncthreads();
      for (int l = threadIdx.x; l < N2; l += blockDim.x) {
        const int a = l % N, b = l / N, I = ex * P + a, J = ey * P + b;
        if (DIR && bnd2(m, I, J)) continue;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) s += sDB[k * N + a] * s0[k + N * b] + sDB[k * N + b] * s1[a + N * k];
        atomicAdd(v + I + (long long)m.Mx * J, s);
      }
    } else {
      for (int q = threadIdx.x; q < N2; q += blockDim.x) {   // x passes: t0 = DB_x u, t1 = B_x u  [i + N b]
        const int i = q % N, b = q / N;
        double d = 0.0, c = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) {
          d += sDB[i * N + a] * su[a + N * b];
          c += sB[i * N + a] * su[a + N * b];
        }
        t0[q] = d;
        t1[q] = c;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < N2; q += blockDim.x) {   // y passes and the factors at (i, j)
        const int i = q % N, j = q / N;
        double g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) {
          g0 += sB[j * N + b] * t0[i + N * b];
          g1 += sDB[j * N + b] * t1[i + N * b];
        }
        s0[q] = Ge[q] * g0 + Ge[N2 + q] * g1;
        s1[q] = Ge[N2 + q] * g0 + Ge[2 * N2 + q] * g1;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < N2; q += blockDim.x) {   // transposed x passes  [a + N j]
        const int a = q % N, j = q / N;
        double d = 0.0, c = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          d += sDB[i * N + a] * s0[i + N * j];
          c += sB[i * N + a] * s1[i + N * j];
        }
        t0[q] = d;
        t1[q] = c;
      }
      __syncthreads();
      for (int l = threadIdx.x; l < N2; l += blockDim.x) {
        const int a = l % N, b = l / N, I = ex * P + a, J = ey * P + b;
        if (DIR && bnd2(m, I, J)) continue;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s += sB[j * N + b] * t0[a + N * j] + sDB[j * N + b] * t1[a + N * j];
        atomicAdd(v + I + (long long)m.Mx * J, s);
      }
    }
  }
}

// element diagonal d(a,b) = sum_q grad phi_ab(q)^T G_q grad phi_ab(q), added on interior nodes (bc 0)
template <int P, int Q>
__global__ void __launch_bounds__(128) k_diag2d(MeshDev m, int bc, const double* __restrict__ G, double* d) {
  constexpr int N = P + 1, N2 = N * N;
  __shared__ double sB[N2], sDB[N2], sw[N], sx[N];
  load_tables2<P, Q>(sB, sDB, sw, sx);
  __syncthreads();
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    const int ex = (int)(e % m.nex), ey = (int)(e / m.nex);
    const double* Ge = G + e * 3 * N2;
    for (int l = threadIdx.x; l < N2; l += blockDim.x) {
      const int a = l % N, b = l / N, I = ex * P + a, J = ey * P + b;
      if (bc == 0 && bnd2(m, I, J)) continue;
      double s = 0.0;
      for (int j = 0; j < N; ++j)
        for (int i = 0; i < N; ++i) {
          const int q = i + N * j;
          const double gx = sDB[i * N + a] * sB[j * N + b], gy = sB[i * N + a] * sDB[j * N + b];
          s += Ge[q] * gx * gx + 2.0 * Ge[N2 + q] * gx * gy + Ge[2 * N2 + q] * gy * gy;
        }
      atomicAdd(d + I + (long long)m.Mx * J, s);
    }
  }
}

// load vector of u* = sin(pi x) sin(pi y): b(a,b) = sum_q phi_ab(q) w_q detJ_q f(x_q),
// f = 2 pi^2 mu u* - grad mu . grad u* (P:376); interior nodes
template <int P, int Q>
__global__ void __launch_bounds__(128) k_load2d(MeshDev m, double* f) {
  constexpr int N = P + 1, N2 = N * N;
  __shared__ double sB[N2], sDB[N2], sw[N], sx[N], sX[2 * N2], sF[N2];
  load_tables2<P, Q>(sB, sDB, sw, sx);
  const double pi = 3.14159265358979323846;
  for (long long e = blockIdx.x; e < m.E; e += gridDim.x) {
    const int ex = (int)(e % m.nex), ey = (int)(e / m.nex);
    __syncthreads();
    nodes2<P>(m, sx, ex, ey, sX);
    __syncthreads();
    for (int q = threadIdx.x; q < N2; q += blockDim.x) {
      const int i = q % N, j = q / N;
      double J[2][2], xq[2];
      jac2<P>(sX, sB, sDB, i, j, J, xq);
      const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      const double x = xq[0], y = xq[1];
      const double us = sinpi(x) * sinpi(y);
      const double gu0 = pi * cospi(x) * sinpi(y), gu1 = pi * sinpi(x) * cospi(y);
      const double mu = mu2(m, x, y);
      double gm[2];
      mu2_grad(m, x, y, mu, gm);
      sF[q] = sw[i] * sw[j] * det * (2.0 * pi * pi * mu * us - (gm[0] * gu0 + gm[1] * gu1));
    }
    __syncthreads();
    for (int l = threadIdx.x; l < N2; l += blockDim.x) {
      const int a = l % N, b = l / N, I = ex * P + a, J = ey * P + b;
      if (bnd2(m, I, J)) continue;
      double s = 0.0;
      for (int j = 0; j < N; ++j)
        for (int i = 0; i < N; ++i) s += sB[i * N + a] * sB[j * N + b] * sF[i + N * j];
      atomicAdd(f + I + (long long)m.Mx * J, s);
    }
  }
}

// ------------------------------------------------------------------------------------------ launchers

static unsigned grid2(long long E) {
  long long b = E;
  if (b > 148LL * 16) b = 148LL * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

#define SFMG_2D_DISPATCH(p, F, ...)                                                              \
  switch (p) {                                                                                   \
    case 1: return F<1>(__VA_ARGS__);   case 2: return F<2>(__VA_ARGS__);                        \
    case 3: return F<3>(__VA_ARGS__);   case 4: return F<4>(__VA_ARGS__);                        \
    case 5: return F<5>(__VA_ARGS__);   case 6: return F<6>(__VA_ARGS__);                        \
    case 7: return F<7>(__VA_ARGS__);   case 8: return F<8>(__VA_ARGS__);                        \
    case 9: return F<9>(__VA_ARGS__);   case 10: return F<10>(__VA_ARGS__);                      \
    case 11: return F<11>(__VA_ARGS__); case 12: return F<12>(__VA_ARGS__);                      \
    case 13: return F<13>(__VA_ARGS__); case 14: return F<14>(__VA_ARGS__);                      \
    case 15: return F<15>(__VA_ARGS__); case 16: return F<16>(__VA_ARGS__);                      \
  }                                                                                              \
  return cudaErrorInvalidValue;

template <int P>
static cudaError_t geometry2d_p(const MeshDev& m, double* G, int* bad, cudaStream_t s) {
  if (m.quad) k_geometry2d<P, 1><<<grid2(m.E), 128, 0, s>>>(m, G, bad);
  else k_geometry2d<P, 0><<<grid2(m.E), 128, 0, s>>>(m, G, bad);
  return cudaGetLastError();
}
cudaError_t launch_geometry_2d(const MeshDev& m, double* G, int* bad, cudaStream_t s) {
  cudaError_t e = upload_2d_tables(m.p, m.quad);
  if (e) return e;
  SFMG_2D_DISPATCH(m.p, geometry2d_p, m, G, bad, s)
}

template <int P>
static cudaError_t apply2d_p(const MeshDev& m, int bc, const double* G, const double* u, double* v, cudaStream_t s) {
  if (m.quad) {
    if (bc == 0) k_apply2d<P, 1, true><<<grid2(m.E), 128, 0, s>>>(m, G, u, v);
    else k_apply2d<P, 1, false><<<grid2(m.E), 128, 0, s>>>(m, G, u, v);
  } else {
    if (bc == 0) k_apply2d<P, 0, true><<<grid2(m.E), 128, 0, s>>>(m, G, u, v);
    else k_apply2d<P, 0, false><<<grid2(m.E), 128, 0, s>>>(m, G, u, v);
  }
  return cudaGetLastError();
}
cudaError_t launch_apply_2d(const MeshDev& m, int bc, const double* G, const double* u, double* v, cudaStream_t s) {
  SFMG_2D_DISPATCH(m.p, apply2d_p, m, bc, G, u, v, s)
}

template <int P>
static cudaError_t diag2d_p(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s) {
  if (m.quad) k_diag2d<P, 1><<<grid2(m.E), 128, 0, s>>>(m, bc, G, d);
  else k_diag2d<P, 0><<<grid2(m.E), 128, 0, s>>>(m, bc, G, d);
  return cudaGetLastError();
}
cudaError_t launch_diag_2d(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s) {
  SFMG_2D_DISPATCH(m.p, diag2d_p, m, bc, G, d, s)
}

template <int P>
static cudaError_t load2d_p(const MeshDev& m, double* f, cudaStream_t s) {
  if (m.quad) k_load2d<P, 1><<<grid2(m.E), 128, 0, s>>>(m, f);
  else k_load2d<P, 0><<<grid2(m.E), 128, 0, s>>>(m, f);
  return cudaGetLastError();
}
cudaError_t launch_load_2d(const MeshDev& m, double* f, cudaStream_t s) {
  SFMG_2D_DISPATCH(m.p, load2d_p, m, f, s)
}

}  // namespace sfmg

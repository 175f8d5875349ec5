// Multigrid transfer kernels for sm_100a (eq. (7)): p-transfer
// p/2 <-> p on one element grid, and (NEXT-1) h-transfer at p = 1 between nested element grids.
//
// Prolongation p/2 -> p on one element grid: P_gJ = phi^{p/2}_J(xi(g)); per element this is the
// tensor contraction u_f(i,j,k) = sum_{abc} I[i][a] I[j][b] I[k][c] u_c(a,b,c) with the 1-D
// interpolation matrix I[i][a] = ell^{p/2}_a(xhat^p_i), evaluated sum-factorised (x, y, z passes
// through shared memory).  P0 = M_f P M_c: coarse boundary values are read as 0 and fine boundary
// rows are not written (add) or written as 0 (overwrite).  Every fine node is written once, by its
// canonical (lowest-index) element, so no atomics are needed.
// Restriction is the exact transpose: each element contracts the fine values it owns with I^T
// and adds the coarse result into r_c (fp64 RED), coarse boundary rows excluded (R12).
#include "sfmg_internal.h"

namespace sfmg {

__constant__ double c_I[8][17 * 9];   // c_I[pc-1][i*(pc+1)+a], fine order 2 pc
static OncePerDevice g_interp_uploaded[9];

cudaError_t upload_interp_tables(int pc, cudaStream_t s) {
  (void)s;
  if (pc < 1 || pc > 8) return cudaErrorInvalidValue;
  return g_interp_uploaded[pc].run([&]() -> cudaError_t {
  std::vector<double> I = make_interp(pc, 2 * pc);
  cudaError_t e = cudaMemcpyToSymbol(c_I, I.data(), sizeof(double) * I.size(), sizeof(double) * 17 * 9 * (pc - 1));
  if (e) return e;
  return cudaSuccess;
  });
}

// element index -> (ex, ey, ez); E < 2^31 (checked at level creation), so 32-bit unsigned
// division (a 64-bit divide costs ~5x more instructions and sits in every apply thread's loop)
__device__ __forceinline__ void ecoords(const MeshDev& m, long long e, int& ex, int& ey, int& ez) {
  const unsigned ue = (unsigned)e;
  const unsigned t = ue / (unsigned)m.nex;
  ex = (int)(ue - t * (unsigned)m.nex);
  ez = (int)(t / (unsigned)m.ney);
  ey = (int)(t - (unsigned)ez * (unsigned)m.ney);
}

template <int PC>
struct XferCfg {
  static constexpr int PF = 2 * PC, NC = PC + 1, NF = PF + 1;
  static constexpr int NC3 = NC * NC * NC, NF3 = NF * NF * NF;
  static constexpr int T1 = NF * NC * NC, T2 = NF * NF * NC;      // prolong intermediates
  static constexpr int R1 = NC * NF * NF, R2 = NC * NC * NF;      // restrict intermediates
  static constexpr size_t SMEM_P = sizeof(double) * (NC3 + T1 + T2 + NF * NC);   // + I (k_prolong)
  static constexpr size_t SMEM_R = sizeof(double) * NF3;   // the three passes run in place
};

// Prolongation: thread per output value in each pass, I copied to shared memory (a thread-dependent
// row index into __constant__ memory serialises the warp).  Restriction: one thread per 1-D line in
// each pass; every thread runs the same unrolled loop over the line's outputs, so each I[i][a] is a
// compile-time __constant__ operand (uniform across the warp) and each input is loaded once per line
// (measured, cold: restrict<8> 43 -> 31 us; the line form of the prolongation needs 167 registers and
// is slower, 53 vs 35 us).
constexpr int kXferThreads = 320;

template <int PC>
__global__ void __launch_bounds__(256) k_prolong(MeshDev mc, MeshDev mf, const double* __restrict__ uc,
                                                 double* __restrict__ uf, int add) {
  using C = XferCfg<PC>;
  constexpr int NC = C::NC, NF = C::NF, PF = C::PF;
  extern __shared__ double sm[];
  double* sc = sm;             // [c][b][a]
  double* t1 = sc + C::NC3;    // [c][b][i]
  double* t2 = t1 + C::T1;     // [c][j][i]
  double* I = t2 + C::T2;      // [i][a]
  for (int l = threadIdx.x; l < NF * NC; l += blockDim.x) I[l] = c_I[PC - 1][l];
  const long long e = blockIdx.x;
  int ex, ey, ez;
  ecoords(mf, e, ex, ey, ez);
  for (int l = threadIdx.x; l < C::NC3; l += blockDim.x) {
    const int a = l % NC, b = (l / NC) % NC, c = l / (NC * NC);
    const int I0 = ex * PC + a, J0 = ey * PC + b, K0 = ez * PC + c;
    const bool bnd = I0 == 0 || I0 == mc.Mx - 1 || J0 == 0 || J0 == mc.My - 1 || K0 == 0 || K0 == mc.Mz - 1;
    sc[l] = bnd ? 0.0 : uc[I0 + (long long)mc.Mx * (J0 + (long long)mc.My * K0)];
  }
  __syncthreads();
  for (int l = threadIdx.x; l < C::T1; l += blockDim.x) {
    const int i = l % NF, r = l / NF;     // r = b + NC c
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < NC; ++a) s += I[i * NC + a] * sc[a + NC * r];
    t1[l] = s;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < C::T2; l += blockDim.x) {
    const int i = l % NF, j = (l / NF) % NF, c = l / (NF * NF);
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < NC; ++b) s += I[j * NC + b] * t1[i + NF * (b + NC * c)];
    t2[l] = s;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < C::NF3; l += blockDim.x) {
    const int i = l % NF, j = (l / NF) % NF, k = l / (NF * NF);
    if ((i == 0 && ex > 0) || (j == 0 && ey > 0) || (k == 0 && ez > 0)) continue;   // not the owner
    const int I0 = ex * PF + i, J0 = ey * PF + j, K0 = ez * PF + k;
    const bool bnd = I0 == 0 || I0 == mf.Mx - 1 || J0 == 0 || J0 == mf.My - 1 || K0 == 0 || K0 == mf.Mz - 1;
    const long long g = I0 + (long long)mf.Mx * (J0 + (long long)mf.My * K0);
    if (bnd) {
      if (!add) uf[g] = 0.0;
      continue;
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) s += I[k * NC + c] * t2[i + NF * (j + NF * c)];
    // add: one fp64 RED per node (each fine node has exactly one owner, so the result is the same single
    // rounding of uf + s as a load-add-store, without the dependent L2 round trip per output:
    // k_prolong<8> 36 -> see profiles/r02_experiments.md)
    if (add) atomicAdd(uf + g, s); else uf[g] = s;
  }
}

template <int PC>
__global__ void __launch_bounds__(kXferThreads) k_restrict(MeshDev mc, MeshDev mf, const double* __restrict__ rf,
                                                           double* __restrict__ rc) {
  using C = XferCfg<PC>;
  constexpr int NC = C::NC, NF = C::NF, PF = C::PF;
  extern __shared__ double sm[];
  // One array, the passes in place (a line is read and rewritten by one thread): fine values [k][j][i],
  // after x the coarse a sits in slot i = a, after y the coarse b in slot j = b.  39 KB at pc = 8, so
  // five blocks per SM and all 512 blocks of the config-5 fine level resident at once (the three-array
  // form held 71 KB: 3 blocks per SM, two waves).
  double* sf = sm;
  const double* I = c_I[PC - 1];
  const long long e = blockIdx.x;
  int ex, ey, ez;
  ecoords(mf, e, ex, ey, ez);
  for (int l = threadIdx.x; l < C::NF3; l += blockDim.x) {
    const int i = l % NF, j = (l / NF) % NF, k = l / (NF * NF);
    double v = 0.0;
    if (!((i == 0 && ex > 0) || (j == 0 && ey > 0) || (k == 0 && ez > 0))) {
      const int I0 = ex * PF + i, J0 = ey * PF + j, K0 = ez * PF + k;
      const bool bnd = I0 == 0 || I0 == mf.Mx - 1 || J0 == 0 || J0 == mf.My - 1 || K0 == 0 || K0 == mf.Mz - 1;
      if (!bnd) v = rf[I0 + (long long)mf.Mx * (J0 + (long long)mf.My * K0)];
    }
    sf[l] = v;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < NF * NF; r += blockDim.x) {   // x: fine line (j, k) -> NC values
    double L[NF];
#pragma unroll
    for (int i = 0; i < NF; ++i) L[i] = sf[i + NF * r];
#pragma unroll
    for (int a = 0; a < NC; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < NF; ++i) acc = fma(I[i * NC + a], L[i], acc);
      sf[a + NF * r] = acc;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < NC * NF; r += blockDim.x) {   // y: line (a, k) over j -> b
    const int a = r % NC, k = r / NC;
    double L[NF];
#pragma unroll
    for (int j = 0; j < NF; ++j) L[j] = sf[a + NF * (j + NF * k)];
#pragma unroll
    for (int b = 0; b < NC; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NF; ++j) acc = fma(I[j * NC + b], L[j], acc);
      sf[a + NF * (b + NF * k)] = acc;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < NC * NC; r += blockDim.x) {   // z: line (a, b) over k -> c, RED
    const int a = r % NC, b = r / NC;
    const int I0 = ex * PC + a, J0 = ey * PC + b;
    if (I0 == 0 || I0 == mc.Mx - 1 || J0 == 0 || J0 == mc.My - 1) continue;
    double L[NF];
#pragma unroll
    for (int k = 0; k < NF; ++k) L[k] = sf[a + NF * (b + NF * k)];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int K0 = ez * PC + c;
      if (K0 == 0 || K0 == mc.Mz - 1) continue;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NF; ++k) acc = fma(I[k * NC + c], L[k], acc);
      atomicAdd(rc + I0 + (long long)mc.Mx * (J0 + (long long)mc.My * K0), acc);
    }
  }
}

template <int PC>
static cudaError_t prolong_p(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                             cudaStream_t s) {
  using C = XferCfg<PC>;
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_prolong<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_P);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  k_prolong<PC><<<(unsigned)mf.E, 256, C::SMEM_P, s>>>(mc, mf, uc, uf, add);
  return cudaGetLastError();
}

template <int PC>
static cudaError_t restrict_p(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s) {
  using C = XferCfg<PC>;
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_restrict<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_R);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  cudaError_t e = cudaMemsetAsync(rc, 0, sizeof(double) * mc.N, s);
  if (e) return e;
  k_restrict<PC><<<(unsigned)mf.E, kXferThreads, C::SMEM_R, s>>>(mc, mf, rf, rc);
  return cudaGetLastError();
}

cudaError_t launch_prolong(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                           cudaStream_t s) {
  switch (mc.p) {
    case 1: return prolong_p<1>(mc, mf, uc, uf, add, s);
    case 2: return prolong_p<2>(mc, mf, uc, uf, add, s);
    case 3: return prolong_p<3>(mc, mf, uc, uf, add, s);
    case 4: return prolong_p<4>(mc, mf, uc, uf, add, s);
    case 5: return prolong_p<5>(mc, mf, uc, uf, add, s);
    case 6: return prolong_p<6>(mc, mf, uc, uf, add, s);
    case 7: return prolong_p<7>(mc, mf, uc, uf, add, s);
    case 8: return prolong_p<8>(mc, mf, uc, uf, add, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_restrict(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s) {
  switch (mc.p) {
    case 1: return restrict_p<1>(mc, mf, rf, rc, s);
    case 2: return restrict_p<2>(mc, mf, rf, rc, s);
    case 3: return restrict_p<3>(mc, mf, rf, rc, s);
    case 4: return restrict_p<4>(mc, mf, rf, rc, s);
    case 5: return restrict_p<5>(mc, mf, rf, rc, s);
    case 6: return restrict_p<6>(mc, mf, rf, rc, s);
    case 7: return restrict_p<7>(mc, mf, rf, rc, s);
    case 8: return restrict_p<8>(mc, mf, rf, rc, s);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
// h-transfer at p = 1 between nested element grids (fine ne = 2 coarse ne; eq. (7) across
// meshes; nesting in reference-lattice coordinates, R25).  On the p = 1 lattices the
// coarse trilinear basis evaluated at the fine nodes gives, per axis, weight 1 for fine index
// I = 2 Ic and 1/2 for I = 2 Ic +- 1.  Both directions are gathers (thread per output node): no
// atomics, deterministic.  P0 = M_f P M_c (R12).

struct HW {   // the (<= 2) coarse indices and weights of one fine lattice index
  int i0, i1;
  double w0, w1;
};
__device__ __forceinline__ HW hweights(int I) {
  HW h;
  if ((I & 1) == 0) { h.i0 = h.i1 = I >> 1; h.w0 = 1.0; h.w1 = 0.0; }
  else { h.i0 = (I - 1) >> 1; h.i1 = (I + 1) >> 1; h.w0 = h.w1 = 0.5; }
  return h;
}

__global__ void k_prolong_h(MeshDev mc, MeshDev mf, const double* __restrict__ uc, double* __restrict__ uf,
                            int add) {
  const long long n = mf.N;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    const int I = (int)(g % mf.Mx), J = (int)((g / mf.Mx) % mf.My), K = (int)(g / ((long long)mf.Mx * mf.My));
    if (I == 0 || I == mf.Mx - 1 || J == 0 || J == mf.My - 1 || K == 0 || K == mf.Mz - 1) {
      if (!add) uf[g] = 0.0;
      continue;
    }
    const HW hx = hweights(I), hy = hweights(J), hz = hweights(K);
    const int ix[2] = {hx.i0, hx.i1}, iy[2] = {hy.i0, hy.i1}, iz[2] = {hz.i0, hz.i1};
    const double wx[2] = {hx.w0, hx.w1}, wy[2] = {hy.w0, hy.w1}, wz[2] = {hz.w0, hz.w1};
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const double w = wx[a] * wy[b] * wz[c];
          const int Ic = ix[a], Jc = iy[b], Kc = iz[c];
          if (w == 0.0 || Ic == 0 || Ic == mc.Mx - 1 || Jc == 0 || Jc == mc.My - 1 || Kc == 0 || Kc == mc.Mz - 1)
            continue;   // M_c: coarse boundary values read as zero
          s += w * uc[Ic + (long long)mc.Mx * (Jc + (long long)mc.My * Kc)];
        }
    if (add) uf[g] += s; else uf[g] = s;
  }
}

__global__ void k_restrict_h(MeshDev mc, MeshDev mf, const double* __restrict__ rf, double* __restrict__ rc) {
  const long long n = mc.N;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    const int I = (int)(g % mc.Mx), J = (int)((g / mc.Mx) % mc.My), K = (int)(g / ((long long)mc.Mx * mc.My));
    if (I == 0 || I == mc.Mx - 1 || J == 0 || J == mc.My - 1 || K == 0 || K == mc.Mz - 1) {
      rc[g] = 0.0;
      continue;
    }
    double s = 0.0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int If = 2 * I + dx, Jf = 2 * J + dy, Kf = 2 * K + dz;
          if (If == 0 || If == mf.Mx - 1 || Jf == 0 || Jf == mf.My - 1 || Kf == 0 || Kf == mf.Mz - 1) continue;
          const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);   // M_f r_f
          s += w * rf[If + (long long)mf.Mx * (Jf + (long long)mf.My * Kf)];
        }
    rc[g] = s;
  }
}

static unsigned hgrid(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148LL * 16) b = 148LL * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_prolong_h(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                             cudaStream_t s) {
  if (mc.p != 1 || mf.p != 1) return cudaErrorInvalidValue;
  k_prolong_h<<<hgrid(mf.N), 256, 0, s>>>(mc, mf, uc, uf, add);
  return cudaGetLastError();
}

cudaError_t launch_restrict_h(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s) {
  if (mc.p != 1 || mf.p != 1) return cudaErrorInvalidValue;
  k_restrict_h<<<hgrid(mc.N), 256, 0, s>>>(mc, mf, rf, rc);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// h-transfer at any order p (NEXT-4: "high-order restriction and prolongation").  Fine
// element (ex, ey, ez) is child (ex & 1, ey & 1, ez & 1) of coarse element (ex/2, ey/2, ez/2), so
// per element P is the tensor contraction u_f(i,j,k) = sum_{abc} H_sx[i][a] H_sy[j][b] H_sz[k][c]
// u_c(a,b,c) with the child matrices H_s = make_h_interp(p, s) -- the same sum-factorised x, y, z
// passes as the p-transfer; canonical owners write (prolong), restriction is the exact transpose
// with fp64 REDs into the coarse element.  P0 = M_f P M_c (R12).

constexpr int hOffset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += 2 * (q + 1) * (q + 1);
  return s;
}
__constant__ double c_H[hOffset(17)];   // per order: H_0 then H_1, [i][a]
static OncePerDevice g_h_uploaded[17];

cudaError_t upload_h_tables(int p) {
  if (p < 1 || p > 16) return cudaErrorInvalidValue;
  return g_h_uploaded[p].run([&]() -> cudaError_t {
  const int n = p + 1;
  for (int sc = 0; sc < 2; ++sc) {
    std::vector<double> H = make_h_interp(p, sc);
    cudaError_t e = cudaMemcpyToSymbol(c_H, H.data(), sizeof(double) * n * n, sizeof(double) * (hOffset(p) + sc * n * n));
    if (e) return e;
  }
  return cudaSuccess;
  });
}

template <int P>
__device__ __forceinline__ double hmat(int s, int i, int a) {
  return c_H[hOffset(P) + s * (P + 1) * (P + 1) + i * (P + 1) + a];
}

template <int P>
__global__ void __launch_bounds__(256) k_prolong_hp(MeshDev mc, MeshDev mf, const double* __restrict__ uc,
                                                    double* __restrict__ uf, int add) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  extern __shared__ double sm[];
  double* sc = sm;        // [c][b][a]
  double* t1 = sc + N3;   // [c][b][i]
  double* t2 = t1 + N3;   // [c][j][i]
  const long long e = blockIdx.x;
  int ex, ey, ez;
  ecoords(mf, e, ex, ey, ez);
  const int sx = ex & 1, sy = ey & 1, sz = ez & 1;
  const int cx = ex >> 1, cy = ey >> 1, cz = ez >> 1;
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int a = l % N, b = (l / N) % N, c = l / N2;
    const int I0 = cx * P + a, J0 = cy * P + b, K0 = cz * P + c;
    const bool bnd = I0 == 0 || I0 == mc.Mx - 1 || J0 == 0 || J0 == mc.My - 1 || K0 == 0 || K0 == mc.Mz - 1;
    sc[l] = bnd ? 0.0 : uc[I0 + (long long)mc.Mx * (J0 + (long long)mc.My * K0)];
  }
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int i = l % N, r = l / N;
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) s += hmat<P>(sx, i, a) * sc[a + N * r];
    t1[l] = s;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int i = l % N, j = (l / N) % N, c = l / N2;
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < N; ++b) s += hmat<P>(sy, j, b) * t1[i + N * (b + N * c)];
    t2[l] = s;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int i = l % N, j = (l / N) % N, k = l / N2;
    if ((i == 0 && ex > 0) || (j == 0 && ey > 0) || (k == 0 && ez > 0)) continue;   // not the owner
    const int I0 = ex * P + i, J0 = ey * P + j, K0 = ez * P + k;
    const bool bnd = I0 == 0 || I0 == mf.Mx - 1 || J0 == 0 || J0 == mf.My - 1 || K0 == 0 || K0 == mf.Mz - 1;
    const long long g = I0 + (long long)mf.Mx * (J0 + (long long)mf.My * K0);
    if (bnd) {
      if (!add) uf[g] = 0.0;
      continue;
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) s += hmat<P>(sz, k, c) * t2[i + N * (j + N * c)];
    if (add) uf[g] += s; else uf[g] = s;
  }
}

template <int P>
__global__ void __launch_bounds__(256) k_restrict_hp(MeshDev mc, MeshDev mf, const double* __restrict__ rf,
                                                     double* __restrict__ rc) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  extern __shared__ double sm[];
  double* sf = sm;        // [k][j][i]
  double* t1 = sf + N3;   // [k][j][a]
  double* t2 = t1 + N3;   // [k][b][a]
  const long long e = blockIdx.x;
  int ex, ey, ez;
  ecoords(mf, e, ex, ey, ez);
  const int sx = ex & 1, sy = ey & 1, sz = ez & 1;
  const int cx = ex >> 1, cy = ey >> 1, cz = ez >> 1;
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int i = l % N, j = (l / N) % N, k = l / N2;
    double v = 0.0;
    if (!((i == 0 && ex > 0) || (j == 0 && ey > 0) || (k == 0 && ez > 0))) {
      const int I0 = ex * P + i, J0 = ey * P + j, K0 = ez * P + k;
      const bool bnd = I0 == 0 || I0 == mf.Mx - 1 || J0 == 0 || J0 == mf.My - 1 || K0 == 0 || K0 == mf.Mz - 1;
      if (!bnd) v = rf[I0 + (long long)mf.Mx * (J0 + (long long)mf.My * K0)];
    }
    sf[l] = v;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int a = l % N, r = l / N;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s += hmat<P>(sx, i, a) * sf[i + N * r];
    t1[l] = s;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int a = l % N, b = (l / N) % N, k = l / N2;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s += hmat<P>(sy, j, b) * t1[a + N * (j + N * k)];
    t2[l] = s;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += blockDim.x) {
    const int a = l % N, b = (l / N) % N, c = l / N2;
    const int I0 = cx * P + a, J0 = cy * P + b, K0 = cz * P + c;
    const bool bnd = I0 == 0 || I0 == mc.Mx - 1 || J0 == 0 || J0 == mc.My - 1 || K0 == 0 || K0 == mc.Mz - 1;
    if (bnd) continue;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s += hmat<P>(sz, k, c) * t2[a + N * (b + N * k)];
    atomicAdd(rc + I0 + (long long)mc.Mx * (J0 + (long long)mc.My * K0), s);
  }
}

template <int P>
static cudaError_t prolong_hp_p(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                                cudaStream_t s) {
  constexpr size_t smem = sizeof(double) * 3 * (P + 1) * (P + 1) * (P + 1);
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_prolong_hp<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  k_prolong_hp<P><<<(unsigned)mf.E, 256, smem, s>>>(mc, mf, uc, uf, add);
  return cudaGetLastError();
}

template <int P>
static cudaError_t restrict_hp_p(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s) {
  constexpr size_t smem = sizeof(double) * 3 * (P + 1) * (P + 1) * (P + 1);
  static OncePerDevice attr;
  {
    cudaError_t ea = attr.run([&]() -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(k_restrict_hp<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      return cudaSuccess;
    });
    if (ea) return ea;
  }
  cudaError_t e = cudaMemsetAsync(rc, 0, sizeof(double) * mc.N, s);
  if (e) return e;
  k_restrict_hp<P><<<(unsigned)mf.E, 256, smem, s>>>(mc, mf, rf, rc);
  return cudaGetLastError();
}

#define SFMG_HP_CASES(F, ...)                                                             \
  switch (mf.p) {                                                                         \
    case 1: return F<1>(__VA_ARGS__);   case 2: return F<2>(__VA_ARGS__);                 \
    case 3: return F<3>(__VA_ARGS__);   case 4: return F<4>(__VA_ARGS__);                 \
    case 5: return F<5>(__VA_ARGS__);   case 6: return F<6>(__VA_ARGS__);                 \
    case 7: return F<7>(__VA_ARGS__);   case 8: return F<8>(__VA_ARGS__);                 \
    case 9: return F<9>(__VA_ARGS__);   case 10: return F<10>(__VA_ARGS__);               \
    case 11: return F<11>(__VA_ARGS__); case 12: return F<12>(__VA_ARGS__);               \
    case 13: return F<13>(__VA_ARGS__); case 14: return F<14>(__VA_ARGS__);               \
    case 15: return F<15>(__VA_ARGS__); case 16: return F<16>(__VA_ARGS__);               \
  }                                                                                       \
  return cudaErrorInvalidValue;

cudaError_t launch_prolong_hp(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                              cudaStream_t s) {
  if (mc.p != mf.p) return cudaErrorInvalidValue;
  cudaError_t e = upload_h_tables(mf.p);
  if (e) return e;
  SFMG_HP_CASES(prolong_hp_p, mc, mf, uc, uf, add, s)
}

cudaError_t launch_restrict_hp(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s) {
  if (mc.p != mf.p) return cudaErrorInvalidValue;
  cudaError_t e = upload_h_tables(mf.p);
  if (e) return e;
  SFMG_HP_CASES(restrict_hp_p, mc, mf, rf, rc, s)
}

// ------------------------------------------------------------------------------------------
// 2-D transfers (NEXT-2): the same eq. (7) contractions on quadrilaterals, block per fine element.
// KIND 1: p pair (fine order 2 PC, same element grid, matrix c_I); KIND 2: h pair at order PC (fine
// element (ex, ey) is child (ex & 1, ey & 1) of coarse element (ex/2, ey/2), matrices c_H).

template <int PC, int KIND>
struct X2 {
  static constexpr int PF = KIND == 1 ? 2 * PC : PC, NC = PC + 1, NF = PF + 1;
  __device__ static double M(int s, int i, int a) {   // fine index i, coarse index a
    if constexpr (KIND == 1) return c_I[PC - 1][i * NC + a];
    else return hmat<PC>(s, i, a);
  }
};

template <int PC, int KIND>
__global__ void __launch_bounds__(128) k_prolong2d(MeshDev mc, MeshDev mf, const double* __restrict__ uc,
                                                   double* __restrict__ uf, int add) {
  using X = X2<PC, KIND>;
  constexpr int NC = X::NC, NF = X::NF, PF = X::PF;
  __shared__ double sc[NC * NC], t1[NF * NC];
  for (long long e = blockIdx.x; e < mf.E; e += gridDim.x) {
    const int ex = (int)(e % mf.nex), ey = (int)(e / mf.nex);
    const int cx = KIND == 1 ? ex : ex >> 1, cy = KIND == 1 ? ey : ey >> 1;
    const int sx = ex & 1, sy = ey & 1;
    __syncthreads();
    for (int l = threadIdx.x; l < NC * NC; l += blockDim.x) {
      const int a = l % NC, b = l / NC, I = cx * PC + a, J = cy * PC + b;
      const bool bnd = I == 0 || I == mc.Mx - 1 || J == 0 || J == mc.My - 1;
      sc[l] = bnd ? 0.0 : uc[I + (long long)mc.Mx * J];
    }
    __syncthreads();
    for (int l = threadIdx.x; l < NF * NC; l += blockDim.x) {
      const int i = l % NF, b = l / NF;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < NC; ++a) s += X::M(sx, i, a) * sc[a + NC * b];
      t1[l] = s;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < NF * NF; l += blockDim.x) {
      const int i = l % NF, j = l / NF;
      if ((i == 0 && ex > 0) || (j == 0 && ey > 0)) continue;   // not the owner
      const int I = ex * PF + i, J = ey * PF + j;
      const long long g = I + (long long)mf.Mx * J;
      if (I == 0 || I == mf.Mx - 1 || J == 0 || J == mf.My - 1) {
        if (!add) uf[g] = 0.0;
        continue;
      }
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < NC; ++b) s += X::M(sy, j, b) * t1[i + NF * b];
      if (add) uf[g] += s; else uf[g] = s;
    }
  }
}

template <int PC, int KIND>
__global__ void __launch_bounds__(128) k_restrict2d(MeshDev mc, MeshDev mf, const double* __restrict__ rf,
                                                    double* __restrict__ rc) {
  using X = X2<PC, KIND>;
  constexpr int NC = X::NC, NF = X::NF, PF = X::PF;
  __shared__ double sf[NF * NF], t1[NC * NF];
  for (long long e = blockIdx.x; e < mf.E; e += gridDim.x) {
    const int ex = (int)(e % mf.nex), ey = (int)(e / mf.nex);
    const int cx = KIND == 1 ? ex : ex >> 1, cy = KIND == 1 ? ey : ey >> 1;
    const int sx = ex & 1, sy = ey & 1;
    __syncthreads();
    for (int l = threadIdx.x; l < NF * NF; l += blockDim.x) {
      const int i = l % NF, j = l / NF, I = ex * PF + i, J = ey * PF + j;
      const bool own = !((i == 0 && ex > 0) || (j == 0 && ey > 0));
      const bool bnd = I == 0 || I == mf.Mx - 1 || J == 0 || J == mf.My - 1;
      sf[l] = (own && !bnd) ? rf[I + (long long)mf.Mx * J] : 0.0;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < NC * NF; l += blockDim.x) {
      const int a = l % NC, j = l / NC;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < NF; ++i) s += X::M(sx, i, a) * sf[i + NF * j];
      t1[l] = s;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < NC * NC; l += blockDim.x) {
      const int a = l % NC, b = l / NC, I = cx * PC + a, J = cy * PC + b;
      if (I == 0 || I == mc.Mx - 1 || J == 0 || J == mc.My - 1) continue;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NF; ++j) s += X::M(sy, j, b) * t1[a + NC * j];
      atomicAdd(rc + I + (long long)mc.Mx * J, s);
    }
  }
}

static unsigned xgrid2(long long E) {
  long long b = E;
  if (b > 148LL * 16) b = 148LL * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

template <int PC, int KIND>
static cudaError_t xfer2d(const MeshDev& mc, const MeshDev& mf, const double* in, double* out, int add, int dir,
                          cudaStream_t s) {
  if (dir == 0) {
    k_prolong2d<PC, KIND><<<xgrid2(mf.E), 128, 0, s>>>(mc, mf, in, out, add);
  } else {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * mc.N, s);
    if (e) return e;
    k_restrict2d<PC, KIND><<<xgrid2(mf.E), 128, 0, s>>>(mc, mf, in, out);
  }
  return cudaGetLastError();
}

// dir 0: out = P0 in (+= if add); dir 1: out = P0^T in.  kind 1 p pair (coarse p <= 8), 2 h pair.
cudaError_t launch_transfer_2d(const MeshDev& mc, const MeshDev& mf, int kind, int dir, const double* in, double* out,
                               int add, cudaStream_t s) {
  cudaError_t e;
  if (kind == 1) {
    if ((e = upload_interp_tables(mc.p, s))) return e;
    switch (mc.p) {
      case 1: return xfer2d<1, 1>(mc, mf, in, out, add, dir, s);
      case 2: return xfer2d<2, 1>(mc, mf, in, out, add, dir, s);
      case 3: return xfer2d<3, 1>(mc, mf, in, out, add, dir, s);
      case 4: return xfer2d<4, 1>(mc, mf, in, out, add, dir, s);
      case 5: return xfer2d<5, 1>(mc, mf, in, out, add, dir, s);
      case 6: return xfer2d<6, 1>(mc, mf, in, out, add, dir, s);
      case 7: return xfer2d<7, 1>(mc, mf, in, out, add, dir, s);
      case 8: return xfer2d<8, 1>(mc, mf, in, out, add, dir, s);
    }
    return cudaErrorInvalidValue;
  }
  if ((e = upload_h_tables(mc.p))) return e;
  switch (mc.p) {
    case 1: return xfer2d<1, 2>(mc, mf, in, out, add, dir, s);   case 2: return xfer2d<2, 2>(mc, mf, in, out, add, dir, s);
    case 3: return xfer2d<3, 2>(mc, mf, in, out, add, dir, s);   case 4: return xfer2d<4, 2>(mc, mf, in, out, add, dir, s);
    case 5: return xfer2d<5, 2>(mc, mf, in, out, add, dir, s);   case 6: return xfer2d<6, 2>(mc, mf, in, out, add, dir, s);
    case 7: return xfer2d<7, 2>(mc, mf, in, out, add, dir, s);   case 8: return xfer2d<8, 2>(mc, mf, in, out, add, dir, s);
    case 9: return xfer2d<9, 2>(mc, mf, in, out, add, dir, s);   case 10: return xfer2d<10, 2>(mc, mf, in, out, add, dir, s);
    case 11: return xfer2d<11, 2>(mc, mf, in, out, add, dir, s); case 12: return xfer2d<12, 2>(mc, mf, in, out, add, dir, s);
    case 13: return xfer2d<13, 2>(mc, mf, in, out, add, dir, s); case 14: return xfer2d<14, 2>(mc, mf, in, out, add, dir, s);
    case 15: return xfer2d<15, 2>(mc, mf, in, out, add, dir, s); case 16: return xfer2d<16, 2>(mc, mf, in, out, add, dir, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sfmg

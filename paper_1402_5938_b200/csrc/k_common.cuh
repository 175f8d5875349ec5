// Device helpers shared by the operator kernels (k_operator.cu) and the Gauss-quadrature variant
// (k_gauss.cu): geometric-factor layout, element / lattice index arithmetic, the coefficient field
// and the warped node positions (R3, R5, R6), and a block-wide sum.  Product code only.
#pragma once
#include <cstdint>

#include "sfmg_internal.h"

namespace sfmg {

// Layout of the geometric factors, slice-major per element: G[e][k][c][j][i], c in (00,01,02,11,
// 12,22).  An element's factors are one contiguous 48 n^3-byte block (one TMA bulk copy), and a
// k-slice of all six components is one contiguous 48 n^2-byte block.
template <int N>
__device__ __forceinline__ int gofs(int c, int ij, int k) { return k * 6 * N * N + c * N * N + ij; }

// Full offset of G(e, c, ij, k).  For p <= 2 (thread-per-element apply) the factors are stored
// element-interleaved in blocks of 32 elements, [E/32][k][6][n^2][32], so that a warp in which
// lane = element reads every component with one coalesced 256-byte access.
template <int P>
struct GLayout {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr bool kTPE = (P <= 2);
  __host__ __device__ static long long padded_elems(long long E) { return kTPE ? ((E + 31) / 32) * 32 : E; }
  __device__ static long long off(long long e, int c, int ij, int k) {
    if (kTPE) return (((e >> 5) * 6 * N3) + (long long)(k * 6 + c) * N2 + ij) * 32 + (e & 31);
    return e * 6 * N3 + gofs<N>(c, ij, k);
  }
};

// element index -> (ex, ey, ez); E < 2^31 (checked at level creation), so 32-bit unsigned
// division (a 64-bit divide costs ~5x more instructions and sits in every apply thread's loop)
__device__ __forceinline__ void elem_coords(const MeshDev& m, long long e, int& ex, int& ey, int& ez) {
  const unsigned ue = (unsigned)e;
  const unsigned t = ue / (unsigned)m.nex;
  ex = (int)(ue - t * (unsigned)m.nex);
  ez = (int)(t / (unsigned)m.ney);
  ey = (int)(t - (unsigned)ez * (unsigned)m.ney);
}

__device__ __forceinline__ bool lattice_boundary(const MeshDev& m, long long g) {
  unsigned int gi = (unsigned int)g;
  unsigned int I = gi % (unsigned)m.Mx;
  unsigned int r = gi / (unsigned)m.Mx;
  unsigned int J = r % (unsigned)m.My;
  unsigned int K = r / (unsigned)m.My;
  return I == 0 || I == (unsigned)m.Mx - 1 || J == 0 || J == (unsigned)m.My - 1 || (int)K == m.Kb0 ||
         (int)K == m.Kb1;   // z planes: 0 and Mz - 1 in 3-D, none in 2-D
}

// mu at a physical point (R3, R6)
__device__ __forceinline__ double coeff_mu(const MeshDev& m, double x, double y, double z) {
  switch (m.coeff) {
    case 0: return m.c0;
    case 1: return exp(m.c1 * sinpi(2.0 * x) * sinpi(2.0 * y) * sinpi(2.0 * z));
    case 2: return exp10(m.c1 * sinpi(2.0 * x) * sinpi(2.0 * y) * sinpi(2.0 * z));
    case 3: {
      double a = cospi(2.0 * x), b = cospi(2.0 * y), c = cospi(2.0 * z);
      return m.c0 + m.c1 * (a * a + b * b + c * c);
    }
  }
  return 0.0;
}

__device__ __forceinline__ void coeff_grad(const MeshDev& m, double x, double y, double z, double mu,
                                           double g[3]) {
  const double tp = 6.283185307179586476925;
  double sx = sinpi(2.0 * x), sy = sinpi(2.0 * y), sz = sinpi(2.0 * z);
  double cx = cospi(2.0 * x), cy = cospi(2.0 * y), cz = cospi(2.0 * z);
  double dS0 = tp * cx * sy * sz, dS1 = tp * sx * cy * sz, dS2 = tp * sx * sy * cz;
  double f = 0.0;
  switch (m.coeff) {
    case 0: g[0] = g[1] = g[2] = 0.0; return;
    case 1: f = m.c1 * mu; break;
    case 2: f = 2.302585092994045684018 * m.c1 * mu; break;
    case 3:
      g[0] = -tp * m.c1 * sinpi(4.0 * x);
      g[1] = -tp * m.c1 * sinpi(4.0 * y);
      g[2] = -tp * m.c1 * sinpi(4.0 * z);
      return;
  }
  g[0] = f * dS0; g[1] = f * dS1; g[2] = f * dS2;
}

// Physical position of local node (a,b,c) of element (ex,ey,ez): reference-cube lattice point
// then the warp x_i += amp sin(pi X) sin(pi Y) sin(pi Z) (R5).
template <int P>
__device__ __forceinline__ void node_pos(const MeshDev& m, const double* xs, int ex, int ey, int ez,
                                         int a, int b, int c, double X[3]) {
  double Xr = (ex + 0.5 * (xs[a] + 1.0)) / m.nex;
  double Yr = (ey + 0.5 * (xs[b] + 1.0)) / m.ney;
  double Zr = (ez + 0.5 * (xs[c] + 1.0)) / m.nez;
  double s = 0.0;
  if (m.warp == 1) s = m.amp * sinpi(Xr) * sinpi(Yr) * sinpi(Zr);
  X[0] = Xr + s; X[1] = Yr + s; X[2] = Zr + s;
}

// TMA / mbarrier / cp.async helpers (inline PTX).

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// The geometric factors are the one stream read exactly once per apply (48 B per point, ~80 % of the
// bytes); their bulk copies and L2 prefetches carry an L2 evict-first policy so that the streamed
// factors do not push u and the RED target v (each touched by up to 8 elements, at different times)
// out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first_policy())
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes),
               "l"(l2_evict_first_policy())
               : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}


__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  __syncthreads();
  if (ln == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = (blockDim.x + 31) >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

}  // namespace sfmg

// O(N) vector kernels of the solvers (Algorithm 1 lines) and of the power
// iteration (R9).  Reductions are deterministic: a fixed grid of kRedBlocks blocks writes
// per-block partials in a fixed order, and the last block to finish (threadfence + counter)
// sums them in a fixed order and writes the scalars, so results do not depend on scheduling.
#include "sfmg_internal.h"

namespace sfmg {

constexpr int kRedThreads = 256;

__device__ __forceinline__ bool vec_boundary(int Mx, int My, int Kb0, int Kb1, long long g) {
  unsigned int gi = (unsigned int)g;
  unsigned int I = gi % (unsigned)Mx;
  unsigned int r = gi / (unsigned)Mx;
  unsigned int J = r % (unsigned)My;
  unsigned int K = r / (unsigned)My;
  return I == 0 || I == (unsigned)Mx - 1 || J == 0 || J == (unsigned)My - 1 || (int)K == Kb0 || (int)K == Kb1;
}

// Block-level sum of NV values per thread into partials[blockIdx][slot..]; returns true in the
// single thread 0 of the last block, after which finals[] holds the grid sums.
template <int NV>
__device__ bool grid_reduce(double (&v)[NV], const RedScratch& r, double (&finals)[NV]) {
  __shared__ double sh[NV][kRedThreads / 32];
  __shared__ bool last;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < kRedThreads / 32; ++w) s += sh[k][w];
      r.partials[blockIdx.x * kRedSlots + k] = s;
    }
    __threadfence();
    unsigned int t = atomicAdd(r.counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  // last block: fixed-order sum of the partials
  __threadfence();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kRedThreads) s += __ldcg(r.partials + b * kRedSlots + k);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return false;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += sh[k][w];
    finals[k] = s;
  }
  *r.counter = 0u;
  return true;
}

__global__ void __launch_bounds__(kRedThreads) k_dot(RedScratch r, const double* __restrict__ a,
                                                     const double* __restrict__ b, long long n, int slot) {
  double v[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[0] += a[i] * b[i];
  double f[1];
  if (grid_reduce<1>(v, r, f)) r.scalars[slot] = f[0];
}

__global__ void __launch_bounds__(kRedThreads) k_power_sums(RedScratch r, const double* __restrict__ x,
                                                            const double* __restrict__ y,
                                                            const double* __restrict__ dinv, long long n) {
  double v[3] = {0.0, 0.0, 0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double xi = x[i], yi = y[i], di = dinv[i];
    const double z = yi * di;
    v[0] += xi * yi;
    v[1] += xi * xi / di;
    v[2] += z * z;
  }
  double f[3];
  if (grid_reduce<3>(v, r, f)) {
    r.scalars[0] = f[0]; r.scalars[1] = f[1]; r.scalars[2] = f[2];
    r.scalars[3] = f[0] / f[1];
    r.scalars[4] = 1.0 / sqrt(f[2]);
  }
}

__global__ void k_power_norm(int Mx, int My, int Kb0, int Kb1, const double* __restrict__ scal, double* x, double* y,
                             const double* __restrict__ dinv, long long n) {
  const double s = scal[4];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double xn = y[i] * dinv[i] * s;
    x[i] = xn;
    y[i] = vec_boundary(Mx, My, Kb0, Kb1, i) ? xn : 0.0;
  }
}

// splitmix64 (R9, R15): output i of the generator seeded with `seed`
__device__ __forceinline__ double uniform_pm1(unsigned long long seed, unsigned long long i) {
  unsigned long long z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

__global__ void k_power_start(int Mx, int My, int Kb0, int Kb1, unsigned long long seed, double* x, double* y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const bool b = vec_boundary(Mx, My, Kb0, Kb1, i);
    x[i] = b ? 0.0 : uniform_pm1(seed, (unsigned long long)i);
    y[i] = 0.0;
  }
}

__global__ void k_pcg_xr(RedScratch r, double* x, double* rv, const double* __restrict__ p,
                         const double* __restrict__ h, int ia, int ib, int slot, long long n) {
  const double alpha = r.scalars[ia] / r.scalars[ib];
  double v[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = rv[i] - alpha * h[i];
    rv[i] = ri;
    v[0] += ri * ri;
  }
  double f[1];
  if (grid_reduce<1>(v, r, f)) r.scalars[slot] = f[0];
}

// General coarse CG (any order; R13), flag-gated so that batches of iterations can be queued and the
// host polls only between batches.  Scalar slots (kCgc*): ||b||^2, rho = ||r||^2, (p, q), ||r_new||^2,
// beta, flag (0 running, 1 converged, 2 breakdown, 3 max_iter), iterations.  Every block reads the
// same flag / (p, q) at kernel start, so an early return is uniform and never leaves grid_reduce's
// block counter half-counted.
__global__ void k_cgc_start(double* scal) {
  scal[kCgcIt] = 0.0;
  scal[kCgcRho] = scal[kCgcBB];
  scal[kCgcFlag] = (scal[kCgcBB] > 0.0) ? 0.0 : 1.0;
}

__global__ void k_cgc_xr(RedScratch r, double* x, double* rv, const double* __restrict__ p,
                         const double* __restrict__ q, long long n) {
  const double flag = r.scalars[kCgcFlag], pq = r.scalars[kCgcPQ];
  if (flag != 0.0 || !(pq > 0.0)) return;
  const double alpha = r.scalars[kCgcRho] / pq;
  double v[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = rv[i] - alpha * q[i];
    rv[i] = ri;
    v[0] += ri * ri;
  }
  double f[1];
  if (grid_reduce<1>(v, r, f)) r.scalars[kCgcRn] = f[0];
}

__global__ void k_cgc_check(double* scal, double rtol, int maxit) {
  if (scal[kCgcFlag] != 0.0) return;
  if (!(scal[kCgcPQ] > 0.0)) { scal[kCgcFlag] = 2.0; return; }
  const double rn = scal[kCgcRn];
  scal[kCgcBeta] = rn / scal[kCgcRho];
  scal[kCgcRho] = rn;
  scal[kCgcIt] += 1.0;
  if (sqrt(rn) <= rtol * sqrt(scal[kCgcBB])) scal[kCgcFlag] = 1.0;
  else if (scal[kCgcIt] >= (double)maxit) scal[kCgcFlag] = 3.0;
}

__global__ void k_cgc_p(const double* __restrict__ scal, double* p, const double* __restrict__ r, long long n) {
  if (scal[kCgcFlag] != 0.0) return;
  const double beta = scal[kCgcBeta];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

__global__ void k_pcg_p(const double* __restrict__ scal, double* p, const double* __restrict__ z, int ia, int ib,
                        long long n) {
  const double beta = scal[ia] / scal[ib];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

__global__ void k_recip(const double* __restrict__ d, double* dinv, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dinv[i] = 1.0 / d[i];
}
__global__ void k_fill(double* x, double v, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void k_residual(const double* __restrict__ b, const double* __restrict__ y, double* r, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    r[i] = b[i] - y[i];
}
__global__ void k_axpy1(double* x, const double* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] += y[i];
}

// Arnoldi in the D-inner product (R26): scalars[slot] = sum a b / dinv = <a, b>_D
__global__ void __launch_bounds__(kRedThreads) k_dotw(RedScratch r, const double* __restrict__ a,
                                                      const double* __restrict__ b,
                                                      const double* __restrict__ dinv, long long n, int slot) {
  double v[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[0] += a[i] * b[i] / dinv[i];
  double f[1];
  if (grid_reduce<1>(v, r, f)) r.scalars[slot] = f[0];
}
// y -= scalars[slot] x  (Gram-Schmidt step with the coefficient left on the device)
__global__ void k_sub_scaled_dev(const double* __restrict__ scal, int slot, const double* __restrict__ x, double* y,
                                 long long n) {
  const double a = scal[slot];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] -= a * x[i];
}
// y = a x (a * dinv) elementwise: w = D^{-1} (A q) when d = dinv, a = 1
__global__ void k_scale_mul(double a, const double* __restrict__ x, const double* __restrict__ d, double* y,
                            long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i] * (d ? d[i] : 1.0);
}

static int vgrid(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148LL * 16) b = 148LL * 16;
  return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_dot(const RedScratch& r, const double* a, const double* b, long long n, int slot, cudaStream_t s) {
  k_dot<<<kRedBlocks, kRedThreads, 0, s>>>(r, a, b, n, slot);
  return cudaGetLastError();
}
cudaError_t launch_power_step(const MeshDev& m, const RedScratch& r, double* x, double* y, const double* dinv,
                              cudaStream_t s) {
  k_power_sums<<<kRedBlocks, kRedThreads, 0, s>>>(r, x, y, dinv, m.N);
  k_power_norm<<<vgrid(m.N), 256, 0, s>>>(m.Mx, m.My, m.Kb0, m.Kb1, r.scalars, x, y, dinv, m.N);
  return cudaGetLastError();
}
cudaError_t launch_power_start(const MeshDev& m, uint64_t seed, double* x, double* y, cudaStream_t s) {
  k_power_start<<<vgrid(m.N), 256, 0, s>>>(m.Mx, m.My, m.Kb0, m.Kb1, (unsigned long long)seed, x, y, m.N);
  return cudaGetLastError();
}
cudaError_t launch_pcg_xr(const RedScratch& red, double* x, double* r, const double* p, const double* h, int ia,
                          int ib, int slot, long long n, cudaStream_t s) {
  k_pcg_xr<<<kRedBlocks, kRedThreads, 0, s>>>(red, x, r, p, h, ia, ib, slot, n);
  return cudaGetLastError();
}
cudaError_t launch_pcg_p(const RedScratch& red, double* p, const double* z, int ia, int ib, long long n,
                         cudaStream_t s) {
  k_pcg_p<<<vgrid(n), 256, 0, s>>>(red.scalars, p, z, ia, ib, n);
  return cudaGetLastError();
}
cudaError_t launch_recip(const double* d, double* dinv, long long n, cudaStream_t s) {
  k_recip<<<vgrid(n), 256, 0, s>>>(d, dinv, n);
  return cudaGetLastError();
}
cudaError_t launch_fill(double* x, double v, long long n, cudaStream_t s) {
  k_fill<<<vgrid(n), 256, 0, s>>>(x, v, n);
  return cudaGetLastError();
}
cudaError_t launch_copy(const double* a, double* b, long long n, cudaStream_t s) {
  k_copy<<<vgrid(n), 256, 0, s>>>(a, b, n);
  return cudaGetLastError();
}
cudaError_t launch_residual(const double* b, const double* y, double* r, long long n, cudaStream_t s) {
  k_residual<<<vgrid(n), 256, 0, s>>>(b, y, r, n);
  return cudaGetLastError();
}
cudaError_t launch_dotw(const RedScratch& r, const double* a, const double* b, const double* dinv, long long n,
                        int slot, cudaStream_t s) {
  k_dotw<<<kRedBlocks, kRedThreads, 0, s>>>(r, a, b, dinv, n, slot);
  return cudaGetLastError();
}
cudaError_t launch_sub_scaled_dev(const RedScratch& r, int slot, const double* x, double* y, long long n,
                                  cudaStream_t s) {
  k_sub_scaled_dev<<<vgrid(n), 256, 0, s>>>(r.scalars, slot, x, y, n);
  return cudaGetLastError();
}
cudaError_t launch_scale_mul(double a, const double* x, const double* d, double* y, long long n, cudaStream_t s) {
  k_scale_mul<<<vgrid(n), 256, 0, s>>>(a, x, d, y, n);
  return cudaGetLastError();
}
cudaError_t launch_axpy1(double* x, const double* y, long long n, cudaStream_t s) {
  k_axpy1<<<vgrid(n), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

cudaError_t launch_cgc_start(const RedScratch& red, cudaStream_t s) {
  k_cgc_start<<<1, 1, 0, s>>>(red.scalars);
  return cudaGetLastError();
}
cudaError_t launch_cgc_iter_tail(const RedScratch& red, double* x, double* r, double* p, const double* q, long long n,
                                 double rtol, int maxit, cudaStream_t s) {
  k_cgc_xr<<<kRedBlocks, kRedThreads, 0, s>>>(red, x, r, p, q, n);
  k_cgc_check<<<1, 1, 0, s>>>(red.scalars, rtol, maxit);
  k_cgc_p<<<vgrid(n), 256, 0, s>>>(red.scalars, p, r, n);
  return cudaGetLastError();
}

}  // namespace sfmg

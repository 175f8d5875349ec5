// Developer microbenchmark: latency of dependent DFMA chains and of shared-memory loads on one warp,
// and DFMA throughput with k independent chains per thread (cycles per DFMA per warp).
#include <cstdio>
__global__ void chain(double* out, long long* cyc, int k_indep, double a, double b) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  if (k_indep == 1) {
#pragma unroll 1
    for (int it = 0; it < 1024; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r) x[0] = fma(x[0], a, b);
    }
  } else if (k_indep == 4) {
#pragma unroll 1
    for (int it = 0; it < 1024; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c] = fma(x[c], a, b);
    }
  } else if (k_indep == 16) {
#pragma unroll 1
    for (int it = 0; it < 1024; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 16; ++c) x[c] = fma(x[c], a, b);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void lds_lat(double* out, long long* cyc) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) % 1024;
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 4096; ++it) idx = (int)sm[idx];
  long long t1 = clock64();
  out[threadIdx.x] = idx;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h[148];
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 4096);
  for (int k : {1, 4, 16}) {
    for (int warps : {1, 4, 8}) {
      chain<<<1, 32 * warps>>>(out, cyc, k, 1.0000001, 1e-9);
      cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("indep %2d chains/thread, %d warps/block: %.2f cycles per DFMA instruction per warp (chain step)\n", k,
             warps, (double)h[0] / (1024.0 * 8 * k));
    }
  }
  lds_lat<<<1, 32>>>(out, cyc);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 dependent-chain latency (incl. F2I/I2F): %.1f cycles\n", (double)h[0] / 4096.0);
  return 0;
}

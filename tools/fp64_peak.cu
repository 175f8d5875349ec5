// FP64 vector (DFMA) peak of this GPU, measured under sustained load ("the FP64 peak is
// not in MEASURED_PEAKS.json and must be measured on the box with a DFMA-chain microbenchmark").
// Every thread runs CH independent DFMA chains; the grid fills every SM at full occupancy.  Prints one
// JSON line: {"fp64_dfma_tflops": ..., "sm_count": ..., "ms": ...}.  Measurement tool only (not part of
// the library or the hot path).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;          // independent chains per thread (covers the DFMA latency)
constexpr int ITERS = 4096;    // inner iterations per launch

__global__ void __launch_bounds__(256) k_dfma(double* out, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1.2345e300) out[threadIdx.x] = s;   // keeps the chains live; never true
}

int main() {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dfma, 256, 0);
  double* out = nullptr;
  if (cudaMalloc(&out, 256 * sizeof(double)) != cudaSuccess) return 1;
  const int grid = sms * per_sm * 4;   // several waves: sustained, not burst
  const double a = 0.999999999, b = 1e-7;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<grid, 256>>>(out, a, b);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dfma<<<grid, 256>>>(out, a, b);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) return 1;
  const double flops = 2.0 * CH * ITERS * (double)grid * 256 * reps;
  printf("{\"fp64_dfma_tflops\": %.3f, \"sm_count\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f}\n",
         flops / (ms * 1e-3) / 1e12, sms, per_sm, ms);
  cudaFree(out);
  return 0;
}

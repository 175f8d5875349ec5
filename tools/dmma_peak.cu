// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput of this GPU next to the DFMA peak of
// tools/fp64_peak.cu: decides whether the apply's 1-D contractions could move to the tensor pipe
// (north_star: "FP64 tensor cores are used for the contractions only if ncu shows the FP64 pipe is the
// limit").  Measurement tool only (not part of the library or the hot path).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;          // independent accumulator tiles per warp
constexpr int ITERS = 2048;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) k_dmma(double* out, double a, double b) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = threadIdx.x * 1e-9 + i; c[i][1] = 0.5 * i; }
#pragma unroll 2
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345e300) out[threadIdx.x] = s;
}

template <int NW>
static void run(int sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dmma<NW>, NW * 32, 0);
  double* out = nullptr;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int grid = sms * per_sm * 4;
  const double a = 0.999999, b = 1e-9;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dmma<NW><<<grid, NW * 32>>>(out, a, b);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dmma<NW><<<grid, NW * 32>>>(out, a, b);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  // one m8n8k4 = 8*8*4 = 256 FMA = 512 flop per warp instruction
  const double flops = 512.0 * CH * ITERS * (double)grid * NW * reps;
  printf("{\"dmma_m8n8k4_tflops\": %.3f, \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"err\": \"%s\"}\n",
         flops / (ms * 1e-3) / 1e12, NW, per_sm, ms, cudaGetErrorString(err));
  cudaFree(out);
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  run<1>(sms);
  run<4>(sms);
  run<8>(sms);
  return 0;
}

// Dev tool: measured fp64 FMA (DFMA) throughput of this GPU, the denominator
// SURVEY 8(d) asks the complex128 configs to report executed fp64 FLOP/s
// against.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dfma_peak dfma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 1 << 14;

__global__ void dfma_loop(double* out, double b, double c) {
  double a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * kChains * kIters * (double)blocks * threads;
  printf("{\"dfma_tflops\": %.3f, \"sms\": %d, \"ms\": %.4f, \"blocks\": %d, \"threads\": %d}\n",
         flops / best / 1e9, sms, best, blocks, threads);
  return cudaGetLastError() != cudaSuccess;
}

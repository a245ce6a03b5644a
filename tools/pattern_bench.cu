// Dev microbenchmark: HBM bandwidth of the line access patterns the staged
// passes use (8-byte lanes, 16 lanes per 128-byte line), no arithmetic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ld(const float2* p) {
  uint2 r;
  asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ void st(float2* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

// mode 0: sequential copy; mode 1: gather column blocks (read line (cb, row) at cb*16 + row*C),
// write sequentially; mode 2: read sequentially, scatter-write column blocks.
// Each thread handles 16 lines (like the kernels: 16 independent loads in flight).
__global__ void __launch_bounds__(256) pat(const float2* __restrict__ src, float2* __restrict__ dst, int64_t n,
                                           int64_t C, int mode, int64_t nunits, int reps = 1) {
  for (int rep = 0; rep < reps; ++rep) {
  const int lane = threadIdx.x & 15, hw = threadIdx.x >> 4;  // 16 half-warps per CTA
  const int64_t R = n / C;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    // a unit = 256 lines; half-warp hw handles lines u*256 + hw + 16*t
    float2 v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int64_t i = u * 256 + hw + 16 * t;  // line id
      int64_t off;
      if (mode == 6 || mode == 7) {  // consecutive units: same 256 rows, adjacent column blocks (2 or 4)
        const int64_t W = mode == 6 ? 2 : 4, RBK = R / 256;
        const int64_t w = u % W, rb = (u / W) % RBK, cb = (u / W / RBK) * W + w;
        off = cb * 16 + (rb * 256 + hw + 16 * t) * C;
      } else if (mode == 1) off = (i / R) * 16 + (i % R) * C;
      else if (mode >= 3) {  // W = 2^(mode-2) adjacent column blocks of a row read together
        const int W = 1 << (mode - 2);
        const int64_t j = i / W, w = i % W;
        off = ((j / R) * W + w) * 16 + (j % R) * C;
      } else off = i * 16;
      v[t] = ld(src + off + lane);
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int64_t i = u * 256 + hw + 16 * t;
      int64_t off;
      if (mode == 2) off = (i / R) * 16 + (i % R) * C;
      else off = i * 16;
      st(dst + off + lane, v[t]);
    }
  }
  }
}

__device__ __forceinline__ float4 ld4(const float4* p) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
// 16-byte lanes: 8 lanes per 128-byte line; a unit = 512 lines (256 threads x 16 loads / 8)
__global__ void __launch_bounds__(256) pat16(const float2* __restrict__ src, float2* __restrict__ dst, int64_t n,
                                             int64_t C, int mode, int64_t nunits, int W = 1) {
  const int lane = threadIdx.x % (8 * W), grp = threadIdx.x / (8 * W);  // 32/W segment-groups per CTA
  const int64_t R = n / C;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    float4 v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int64_t i = u * (512 / W) + grp + (32 / W) * t;  // segment id
      const int64_t off = mode == 1 ? (i / R) * 16 * W + (i % R) * C : i * 16 * W;
      v[t] = ld4(reinterpret_cast<const float4*>(src + off) + lane);
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int64_t i = u * (512 / W) + grp + (32 / W) * t;
      st4(reinterpret_cast<float4*>(dst + i * 16 * W) + lane, v[t]);
    }
  }
}

int main() {
  const int64_t n = 1ll << 30;
  float2 *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaMemset(b, 0, n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nunits = n / 16 / 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode : {0, 1})
    for (int64_t C : {1ll << 15, 1ll << 12, 1ll << 8})
      for (int occ : {4, 8}) {
        if (C != (1ll << 15)) continue;
        const int grid = sms * occ;
        pat<<<grid, 256>>>(a, b, n, C, mode, nunits);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) pat<<<grid, 256>>>(a, b, n, C, mode, nunits);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3;
        printf("mode=%d C=2^%d ctas/sm=%d: %.3f ms  %.0f GB/s\n", mode, __builtin_ctzll(C), occ, ms,
               2.0 * n * 8 / (ms * 1e-3) / 1e9);
      }
  for (int W : {1, 2, 4})
  for (int mode : {0, 1})
    for (int occ : {4}) {
      const int grid = sms * occ;
      const int64_t nu = n / 16 / 512;
      pat16<<<grid, 256>>>(a, b, n, 1ll << 15, mode, nu, W);
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) pat16<<<grid, 256>>>(a, b, n, 1ll << 15, mode, nu, W);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 3;
      printf("16B lanes segment=%dB mode=%d ctas/sm=%d: %.3f ms  %.0f GB/s\n", 128 * W, mode, occ, ms, 2.0 * n * 8 / (ms * 1e-3) / 1e9);
    }
  // L2-resident copies (32 MB and 16 MB buffers, repeated): L2 read+write bandwidth
  for (int64_t m : {1ll << 22, 1ll << 21, 1ll << 20})
    for (int occ : {4, 8}) {
      const int grid = sms * occ;
      const int64_t nu = m / 16 / 256;
      pat<<<grid, 256>>>(a, b, m, 1ll << 15, 0, nu, 5);
      cudaEventRecord(e0);
      pat<<<grid, 256>>>(a, b, m, 1ll << 15, 0, nu, 50);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 50;
      printf("L2 copy %lld MB ctas/sm=%d: %.4f ms  %.0f GB/s (rd+wr)\n", (long long)(m * 8 >> 20), occ, ms,
             2.0 * m * 8 / (ms * 1e-3) / 1e9);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// L2 bandwidth probe: writes / copies within an L2-resident ring, and the
// staged-pass pattern (HBM->ring, ring->HBM) as one kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__global__ void l2_write(uint4* ring, size_t ring16, size_t total16) {
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total16; i += s) {
    uint4 v = make_uint4(i, 1, 2, 3);
    __stcg(ring + (i % ring16), v);
  }
}
__global__ void l2_copy(uint4* ring, size_t ring16, size_t total16) {
  size_t s = (size_t)gridDim.x * blockDim.x, half = ring16 / 2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total16; i += s) {
    size_t j = i % half;
    __stcg(ring + half + j, __ldcg(ring + j));
  }
}
// staged pattern: even blocks copy HBM->ring, odd blocks ring->HBM
__global__ void staged(const uint4* __restrict__ in, uint4* __restrict__ out, uint4* ring, size_t ring16, size_t n16) {
  size_t nb = gridDim.x / 2, b = blockIdx.x / 2;
  size_t s = nb * blockDim.x;
  if (blockIdx.x & 1) {
    for (size_t i = b * blockDim.x + threadIdx.x; i < n16; i += s) out[i] = __ldcg(ring + (i % ring16));
  } else {
    for (size_t i = b * blockDim.x + threadIdx.x; i < n16; i += s) __stcg(ring + (i % ring16), in[i]);
  }
}
__global__ void copy(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += s) out[i] = in[i];
}
int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  size_t bytes = 4ull << 30, n16 = bytes / 16; uint4 *a, *b, *ring; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&ring, 64 << 20)); cudaMemset(a, 1, bytes);
  for (size_t rb : {16ull << 20, 32ull << 20, 48ull << 20}) {
    size_t r16 = rb / 16;
    l2_write<<<148 * 8, 256>>>(ring, r16, n16); cudaEventRecord(e0);
    l2_write<<<148 * 8, 256>>>(ring, r16, n16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("L2 write ring %zu MB: %.0f GB/s\n", rb >> 20, 1.0 * bytes / ms / 1e6);
    l2_copy<<<148 * 8, 256>>>(ring, r16, n16); cudaEventRecord(e0);
    l2_copy<<<148 * 8, 256>>>(ring, r16, n16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("L2 copy ring %zu MB: %.0f GB/s (rd+wr)\n", rb >> 20, 2.0 * bytes / ms / 1e6);
    staged<<<148 * 8, 256>>>(a, b, ring, r16, n16); cudaEventRecord(e0);
    staged<<<148 * 8, 256>>>(a, b, ring, r16, n16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("staged ring %zu MB: %.2f ms for 4 GiB (HBM rd+wr %.0f GB/s, total L2 %.0f GB/s)\n", rb >> 20, ms, 2.0 * bytes / ms / 1e6, 4.0 * bytes / ms / 1e6);
  }
  copy<<<148 * 8, 256>>>(a, b, n16); cudaEventRecord(e0);
  copy<<<148 * 8, 256>>>(a, b, n16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1); printf("plain copy: %.2f ms (%.0f GB/s)\n", ms, 2.0 * bytes / ms / 1e6);
  return 0;
}

// DRAM locality probe: copy 128-byte column strips of a (rows x cols) matrix
// where concurrently running blocks cover a window of W adjacent strips.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
// each block: strip s (8 x 16B lanes), rows [rb*nrow, (rb+1)*nrow) with row stride `cols` (16B units)
__global__ void win_copy(const uint4* __restrict__ a, uint4* __restrict__ b, int64_t cols, int W, int nrow, int64_t rowblocks) {
  int64_t blk = blockIdx.x;
  int64_t win = blk / (W * rowblocks);
  int64_t rem = blk % (W * rowblocks);
  int64_t rb = rem / W, sw = rem % W;
  int64_t strip = win * W + sw;
  for (int t = threadIdx.x; t < 8 * nrow; t += blockDim.x) {
    int64_t r = rb * nrow + t / 8, c = strip * 8 + t % 8;
    b[r * cols + c] = a[r * cols + c];
  }
}
// runs of L bytes (L = 32,64,128): each thread writes one 16B word; lane groups of L/16 contiguous,
// consecutive groups at stride `gap` (16B units) -- the transposed store pattern
__global__ void run_write(uint4* __restrict__ b, int64_t n16, int Lw, int64_t gap) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t grp = i / Lw, w = i % Lw;
  int64_t ngrp_per_row = gap / Lw;
  int64_t row = grp % (n16 / gap), col = grp / (n16 / gap);
  int64_t addr = row * gap + col * Lw + w;
  if (addr < n16) b[addr] = make_uint4(i, 1, 2, 3);
}
int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  size_t bytes = 4ull << 30; uint4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  int64_t n16 = bytes / 16, cols = 16384;  // 256 KB rows
  int64_t rows = n16 / cols, strips = cols / 8;
  for (int nrow : {16, 64, 256}) for (int W : {1, 2, 4, 8, 16, 32, 64, 2048}) {
    int64_t rowblocks = rows / nrow;
    int64_t blocks = strips * rowblocks;
    win_copy<<<blocks, 128>>>(a, b, cols, W, nrow, rowblocks);
    cudaEventRecord(e0);
    for (int it = 0; it < 3; ++it) win_copy<<<blocks, 128>>>(a, b, cols, W, nrow, rowblocks);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("win_copy 128B strips nrow=%4d W=%5d: %.0f GB/s\n", nrow, W, 2.0 * bytes * 3 / ms / 1e6);
  }
  for (int L : {2, 4, 8, 16, 32}) for (int64_t gap : {16384ll, 65536ll}) {
    int64_t threads = n16; unsigned grid = (unsigned)((threads + 255) / 256);
    run_write<<<grid, 256>>>(b, n16, L, gap);
    cudaEventRecord(e0);
    for (int it = 0; it < 3; ++it) run_write<<<grid, 256>>>(b, n16, L, gap);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("run_write runs=%4d B gap=%lld B: %.0f GB/s\n", L * 16, (long long)gap * 16, 1.0 * bytes * 3 / ms / 1e6);
  }
  return 0;
}

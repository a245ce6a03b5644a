// Dev microbenchmark: memory skeletons of candidate large-FFT pass structures
// on B200, no arithmetic.  N = 2^30 complex64 (8 GiB in, 8 GiB out), viewed as
// a ROWS x COLS matrix of 8-byte elements (COLS = 2^15).  Every kernel moves
// the whole array once (one "pass"); the printed GB/s counts 2*N*8 bytes.
//
//   copy            sequential float4 copy
//   gather F        TMA box {F cols, 256 rows} (strided rows) -> smem -> contiguous STG
//   scatter F       contiguous bulk load -> smem -> strided STG (F-wide segments)
//   both F          TMA strided load -> TMA strided store (pure TMA transpose-free pass)
//   bothstg F       TMA strided load -> strided STG
//   ring            TMA strided load (F=16) -> STG to a per-CTA L2 slot -> bulk load back -> STG out
//   dsm C F NB      cluster of C CTAs: TMA strided loads of a group of F columns x 2^15 rows,
//                   cluster barrier, DSMEM reads of the CTA's slices into registers, strided STG
//   dsmbw C         DSMEM read bandwidth alone (cluster C, full chip)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <type_traits>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));       \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

constexpr int64_t N = int64_t(1) << 30;
constexpr int64_t COLS = int64_t(1) << 15;
constexpr int64_t ROWS = N / COLS;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
          su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma2d_store(const CUtensorMap* m, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0),
               "r"(c1), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void stg16(void* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint4 lds16(const void* p) { return *reinterpret_cast<const uint4*>(p); }

// ---------------------------------------------------------------- copy
__global__ void k_copy(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n16) {
  const uint64_t pf = pol_first();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(s + i), "l"(pf));
    stg16(d + i, v, pf);
  }
}

// ---------------------------------------------------------------- staged TMA kernels
// A "tile" = TB bytes = NBOX boxes of {F, 256}.  Tiles enumerated group-major:
// tile t -> column group cg = t / RB_PER, row block(s) within that group.
struct KP {
  CUtensorMap in, out;  // 2D maps [ROWS][COLS] of u64, box {F, 256}
  const char* src;
  char* dst;
  char* scratch;        // ring: per-CTA L2 slots
  int F, mode;          // mode: 0 gather, 1 scatter, 2 both(TMA store), 3 both(STG), 4 ring
  int W;                // W adjacent column groups interleaved (consecutive tiles: same rows)
  int BR;               // box rows
  int64_t ntiles;
};

template <int STAGES, int TB>
__global__ void __launch_bounds__(256, 1) k_staged(const __grid_constant__ KP p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[STAGES], bar2[STAGES];
  const int tid = threadIdx.x;
  const int F = p.F, SEG = F * 8, BR = p.BR, NBOX = TB / (SEG * BR), W = p.W;
  const int64_t RB_PER = ROWS / BR / NBOX;  // tiles per column group
  auto cg_rb = [&](int64_t t, int64_t& cg, int64_t& rb) {
    const int64_t w = t % W, rest = t / W;
    rb = rest % RB_PER;
    cg = (rest / RB_PER) * W + w;
  };
  const uint64_t pf = pol_first(), pl = pol_last();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mb_init(&bar[s], 1);
      mb_init(&bar2[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t my0 = blockIdx.x, step = gridDim.x;
  auto tile_of = [&](int64_t k) { return my0 + k * step; };
  const int64_t nmine = (p.ntiles - my0 + step - 1) / step;
  auto issue = [&](int64_t k) {  // thread 0
    const int64_t t = tile_of(k);
    const int s = (int)(k % STAGES);
    unsigned char* buf = sm + (size_t)s * TB;
    mb_expect(&bar[s], TB);
    if (p.mode == 1) {
      bulk_g2s(buf, p.src + t * TB, TB, &bar[s], pf);
    } else {
      int64_t cg, rb;
      cg_rb(t, cg, rb);
      for (int b = 0; b < NBOX; ++b)
        tma2d(buf + b * SEG * BR, &p.in, (int)(cg * F), (int)((rb * NBOX + b) * BR), &bar[s], pf);
    }
  };
  if (tid == 0)
    for (int64_t k = 0; k < STAGES - 1 && k < nmine; ++k) issue(k);
  // ring: second buffer set (STAGES more tiles) for the L2 read-back
  unsigned char* rb_sm = sm + (size_t)STAGES * TB;
  char* slotbase = p.scratch + (size_t)blockIdx.x * STAGES * TB;
  for (int64_t k = 0; k < nmine; ++k) {
    const int s = (int)(k % STAGES);
    const uint32_t par = (uint32_t)((k / STAGES) & 1);
    if (tid == 0 && k + STAGES - 1 < nmine) {
      // the stage (k-1) % STAGES was released by the barrier at the end of iteration k-1
      if (p.mode == 2) bulk_wait_read<0>();
      issue(k + STAGES - 1);
    }
    mb_wait(&bar[s], par);
    unsigned char* buf = sm + (size_t)s * TB;
    const int64_t t = tile_of(k);
    if (p.mode == 0) {
      for (int i = tid; i < TB / 16; i += 256) stg16(p.dst + t * TB + i * 16, lds16(buf + i * 16), pf);
    } else if (p.mode == 1 || p.mode == 3) {
      // strided STG: tile t -> (cg, rows); element (row r, col j) of box b at buf[b][r][j]
      int64_t cg, rbk;
      cg_rb(t, cg, rbk);
      const int per_row = SEG / 16;
      for (int i = tid; i < TB / 16; i += 256) {
        const int b = i / (BR * per_row), r = (i / per_row) % BR, q = i % per_row;
        const int64_t row = (rbk * NBOX + b) * BR + r;
        stg16(p.dst + (row * COLS + cg * F) * 8 + q * 16, lds16(buf + i * 16), pf);
      }
    } else if (p.mode == 2) {
      if (tid == 0) {
        int64_t cg, rbk;
        cg_rb(t, cg, rbk);
        for (int b = 0; b < NBOX; ++b) tma2d_store(&p.out, (int)(cg * F), (int)((rbk * NBOX + b) * BR), buf + b * SEG * BR);
        bulk_commit();
      }
    } else if (p.mode == 4) {
      // HBM tile -> this CTA's L2 slot s (evict_last), then read back and stream out
      char* slot = slotbase + (size_t)s * TB;
      for (int i = tid; i < TB / 16; i += 256) stg16(slot + i * 16, lds16(buf + i * 16), pl);
      __syncthreads();
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mb_expect(&bar2[s], TB);
        bulk_g2s(rb_sm + (size_t)s * TB, slot, TB, &bar2[s], pl);
      }
      // consume the previous read-back (one tile behind)
      if (k > 0) {
        const int64_t kp = k - 1;
        const int sp = (int)(kp % STAGES);
        mb_wait(&bar2[sp], (uint32_t)((kp / STAGES) & 1));
        const int64_t tp = tile_of(kp);
        for (int i = tid; i < TB / 16; i += 256)
          stg16(p.dst + tp * TB + i * 16, lds16(rb_sm + (size_t)sp * TB + i * 16), pf);
      }
    }
    __syncthreads();
  }
  if (p.mode == 4 && nmine > 0) {
    const int64_t kp = nmine - 1;
    const int sp = (int)(kp % STAGES);
    mb_wait(&bar2[sp], (uint32_t)((kp / STAGES) & 1));
    const int64_t tp = tile_of(kp);
    for (int i = tid; i < TB / 16; i += 256) stg16(p.dst + tp * TB + i * 16, lds16(rb_sm + (size_t)sp * TB + i * 16), pf);
  }
  if (p.mode == 2 && tid == 0) bulk_wait_read<0>();
}

// ---------------------------------------------------------------- register-staged, 1-deep prefetch
// The tpass structure: one 64 KB landing buffer per CTA (TMA box {32, 256}),
// tile -> registers (32 x 8 B per thread), barrier, next TMA issued, then a
// synthetic compute delay of `delay` cycles and the stores (contiguous).
__global__ void __launch_bounds__(256, 2) k_regs(const __grid_constant__ KP p, int delay, int nbuf) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  constexpr int TBY = 65536;
  const int64_t RB_PER = ROWS / 256;
  const uint64_t pf = pol_first();
  if (tid == 0) {
    mb_init(&bar[0], 1);
    mb_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t my0 = blockIdx.x, step = gridDim.x;
  const int64_t ntiles = N * 8 / TBY;
  const int64_t nmine = (ntiles - my0 + step - 1) / step;
  auto issue = [&](int64_t k) {
    const int64_t t = my0 + k * step;
    const int b = (int)(k % nbuf);
    const int64_t cg = t / RB_PER, rb = t % RB_PER;
    mb_expect(&bar[b], TBY);
    tma2d(sm + (size_t)b * TBY, &p.in, (int)(cg * 32), (int)(rb * 256), &bar[b], pf);
  };
  if (tid == 0) for (int k = 0; k < nbuf - 1 && k < nmine; ++k) issue(k);
  for (int64_t k = 0; k < nmine; ++k) {
    const int b = (int)(k % nbuf);
    if (tid == 0 && nbuf == 1) issue(k);
    mb_wait(&bar[b], (uint32_t)((k / nbuf) & 1));
    uint4 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = lds16(sm + (size_t)b * TBY + (i * 256 + tid) * 16);
    __syncthreads();
    if (tid == 0 && nbuf > 1 && k + nbuf - 1 < nmine) issue(k + nbuf - 1);
    if (delay > 0) {
      const long long t0 = clock64();
      while (clock64() - t0 < delay) {
      }
    }
    const int64_t t = my0 + k * step;
#pragma unroll
    for (int i = 0; i < 16; ++i) stg16(p.dst + t * TBY + (i * 256 + tid) * 16, v[i], pf);
  }
}

// ---------------------------------------------------------------- cluster / DSMEM skeleton
// Cluster of C CTAs handles one group of F columns x ROWS (=2^15) rows at a time:
// CTA c loads rows [c*ROWS/C, (c+1)*ROWS/C) (boxes of 256 rows) into buffer b,
// cluster barrier; then CTA c reads, from every peer, the peer's rows whose
// (row % C) == c  -- a stand-in for the B-stage slice -- into registers; cluster
// barrier (buffer free); strided STG of the registers.  NB buffers per CTA:
// the loads of the next NB-1 groups are in flight during the exchange.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint4 ld_dsm(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

struct DP {
  CUtensorMap in;
  char* dst;
  int C, F, NB;
  int64_t ngroups;
};

template <int NT, int PER>  // PER = 16-byte words per thread per group
__global__ void __launch_bounds__(NT, 1) k_dsm(const __grid_constant__ DP p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[8];
  const int tid = threadIdx.x;
  const int C = p.C, F = p.F, NB = p.NB, SEG = F * 8;
  const uint32_t cr = cluster_rank();
  const int rows_per = (int)(ROWS / C);        // rows this CTA loads per group
  const int gbytes = rows_per * SEG;           // bytes per CTA per group
  const int nclusters = gridDim.x / C, cl = blockIdx.x / C;
  const uint64_t pf = pol_first();
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mb_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t mine = (p.ngroups - cl + nclusters - 1) / nclusters;
  auto issue = [&](int64_t k) {
    const int64_t g = cl + k * nclusters;
    const int b = (int)(k % NB);
    unsigned char* buf = sm + (size_t)b * gbytes;
    mb_expect(&bar[b], gbytes);
    for (int r0 = 0; r0 < rows_per; r0 += 256)
      tma2d(buf + (size_t)r0 * SEG, &p.in, (int)(g * F), (int)(cr * rows_per + r0), &bar[b], pf);
  };
  if (tid == 0)
    for (int64_t k = 0; k < NB - 1 && k < mine; ++k) issue(k);
  cl_arrive();
  cl_wait();
  for (int64_t k = 0; k < mine; ++k) {
    const int b = (int)(k % NB);
    if (tid == 0 && k + NB - 1 < mine) issue(k + NB - 1);
    mb_wait(&bar[b], (uint32_t)((k / NB) & 1));
    cl_arrive();
    cl_wait();  // every CTA's loads of group k have landed
    // my slice: from peer q, its local rows r with r % C == cr; 16-byte words
    const uint32_t base = su32(sm + (size_t)b * gbytes);
    const int words_row = SEG / 16, slice_rows = rows_per / C;
    const int words_peer = slice_rows * words_row;  // per peer
    uint4 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int w = tid + i * NT;  // < C * words_peer
      const int q = w / words_peer, rw = w % words_peer;
      const int r = (rw / words_row) * C + (int)cr, x = rw % words_row;
      v[i] = ld_dsm(mapa(base + (uint32_t)(r * SEG + x * 16), (uint32_t)q));
    }
    cl_arrive();
    cl_wait();  // buffer b may be refilled
    const int64_t g = cl + k * nclusters;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int w = tid + i * NT;
      const int q = w / words_peer, rw = w % words_peer;
      const int64_t row = (int64_t)q * rows_per + (rw / words_row) * C + cr;
      stg16(p.dst + (row * COLS + g * F) * 8 + (rw % words_row) * 16, v[i], pf);
    }
  }
}

// DSMEM bandwidth alone: every CTA repeatedly reads 64 KB spread over all peers
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_dsmbw(int C, int iters, uint4* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t cr = cluster_rank();
  const int tid = threadIdx.x;
  for (int i = tid; i < 65536 / 16; i += NT) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, cr, 1, 2);
  cl_arrive();
  cl_wait();
  const uint32_t base = su32(sm);
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int w = tid; w < 65536 / 16; w += NT) {
      const uint32_t q = (uint32_t)((w / (65536 / 16 / C) + cr + 1) % C);
      const uint4 x = ld_dsm(mapa(base + (uint32_t)(w * 16), q));
      acc.x ^= x.x;
      acc.y += x.y;
      acc.z ^= x.z;
      acc.w += x.w;
    }
  }
  cl_arrive();
  cl_wait();
  if (acc.x == 0x12345 && acc.y == 7) sink[blockIdx.x] = acc;
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn enc() {
  static EncFn f = nullptr;
  if (!f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    f = (EncFn)p;
  }
  return f;
}
static CUtensorMap map2d(void* base, int F, int boxrows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
  cuuint64_t strides[1] = {(cuuint64_t)(COLS * 8)};
  cuuint32_t box[2] = {(cuuint32_t)F, (cuuint32_t)boxrows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed %d (F=%d)\n", (int)r, F);
    exit(1);
  }
  return m;
}

template <class L>
static double timeit(L launch, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}
static void report(const char* what, double ms) {
  printf("%-28s %8.3f ms  %7.0f GB/s (2*N*8 B)\n", what, ms, 2.0 * N * 8 / (ms * 1e6));
  fflush(stdout);
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char *src, *dst, *scratch;
  CK(cudaMalloc(&src, N * 8));
  CK(cudaMalloc(&dst, N * 8));
  CK(cudaMemset(src, 1, N * 8));
  CK(cudaMemset(dst, 0, N * 8));
  CK(cudaMalloc(&scratch, (size_t)sms * 2 * 8 * 32768));
  const char* only = argc > 1 ? argv[1] : "";
  auto want = [&](const char* k) { return !*only || strstr(only, k); };

  if (want("copy"))
    report("copy", timeit([&] { k_copy<<<sms * 8, 512>>>((const uint4*)src, (uint4*)dst, N / 2); }));

  constexpr int TB = 32768;
  auto staged = [&](int mode, int F, const char* name, auto stc, int W = 1) {
    constexpr int ST = decltype(stc)::value;
    KP p;
    memset(&p, 0, sizeof(p));
    p.W = W;
    p.BR = TB / (F * 8) < 256 ? TB / (F * 8) : 256;
    p.in = map2d(src, F, p.BR);
    p.out = map2d(dst, F, p.BR);
    p.src = src;
    p.dst = dst;
    p.scratch = scratch;
    p.F = F;
    p.mode = mode;
    p.ntiles = N * 8 / TB;
    const int smem = (mode == 4 ? 2 : 1) * ST * TB;
    auto fn = k_staged<ST, TB>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
    char nm[64];
    snprintf(nm, sizeof nm, "%s F=%d (%dB) W=%d st=%d occ=%d", name, F, F * 8, W, ST, occ);
    report(nm, timeit([&] { fn<<<sms * occ, 256, smem>>>(p); }));
  };
  using S3 = std::integral_constant<int, 3>;
  using S6 = std::integral_constant<int, 6>;
  for (int F : {16, 32, 64}) {
    for (int W : {1, 2, 4, 8}) {
      if (F * W > 128) continue;
      if (want("gather")) staged(0, F, "gather", S6{}, W);
      if (want("scatter")) staged(1, F, "scatter", S6{}, W);
      if (want("bothtma")) { staged(2, F, "both-tma", S3{}, W); staged(2, F, "both-tma", S6{}, W); }
      if (want("bothstg")) staged(3, F, "both-stg", S6{}, W);
    }
  }
  if (want("ring")) { staged(4, 16, "ring", S3{}, 1); staged(4, 16, "ring", S3{}, 4); }

  if (want("regs")) {
    KP p;
    memset(&p, 0, sizeof(p));
    p.in = map2d(src, 32, 256);
    p.src = src;
    p.dst = dst;
    for (int nbuf : {1, 2}) {
      const int smem = nbuf * 65536;
      CK(cudaFuncSetAttribute(k_regs, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_regs, 256, smem));
      for (int delay : {0, 1000, 2000, 4000, 6000}) {
        char nm[64];
        snprintf(nm, sizeof nm, "regs nbuf=%d occ=%d delay=%d", nbuf, occ, delay);
        report(nm, timeit([&] { k_regs<<<sms * occ, 256, smem>>>(p, delay, nbuf); }));
      }
    }
  }
  if (want("dsm")) {
    struct Cfg { int C, F, NB; };
    for (Cfg c : {Cfg{8, 4, 3}, Cfg{16, 4, 3}, Cfg{16, 8, 1}, Cfg{8, 8, 1}, Cfg{16, 4, 2}, Cfg{8, 4, 2}, Cfg{16, 2, 4}}) {
      const int rows_per = (int)(ROWS / c.C), gbytes = rows_per * c.F * 8;
      const int smem = gbytes * c.NB;
      if (smem > 227 * 1024) continue;
      DP p;
      memset(&p, 0, sizeof(p));
      p.in = map2d(src, c.F, 256);
      p.dst = dst;
      p.C = c.C;
      p.F = c.F;
      p.NB = c.NB;
      p.ngroups = COLS / c.F;
      constexpr int NT = 512;
      const int per = gbytes / 16 / NT;
      void (*fn)(DP) = per == 4 ? k_dsm<NT, 4> : per == 8 ? k_dsm<NT, 8> : per == 16 ? k_dsm<NT, 16> : per == 2 ? k_dsm<NT, 2> : nullptr;
      if (!fn) { printf("dsm C=%d F=%d: per=%d unsupported\n", c.C, c.F, per); continue; }
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (c.C > 8) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t lc = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c.C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.blockDim = dim3(NT);
      lc.dynamicSmemBytes = smem;
      lc.attrs = at;
      lc.numAttrs = 1;
      int ncl = 0;
      lc.gridDim = dim3(c.C);
      CK(cudaOccupancyMaxActiveClusters(&ncl, fn, &lc));
      lc.gridDim = dim3(ncl * c.C);
      char nm[64];
      snprintf(nm, sizeof nm, "dsm C=%d F=%d NB=%d cl=%d", c.C, c.F, c.NB, ncl);
      report(nm, timeit([&] { CK(cudaLaunchKernelEx(&lc, fn, p)); }));
    }
  }
  if (want("dsmbw")) {
    uint4* sink;
    CK(cudaMalloc(&sink, 4096 * 16));
    for (int C : {2, 4, 8, 16}) {
      constexpr int NT = 512;
      auto fn = k_dsmbw<NT>;
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
      if (C > 8) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t lc = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.blockDim = dim3(NT);
      lc.dynamicSmemBytes = 65536;
      lc.attrs = at;
      lc.numAttrs = 1;
      int ncl = 0;
      lc.gridDim = dim3(C);
      CK(cudaOccupancyMaxActiveClusters(&ncl, fn, &lc));
      lc.gridDim = dim3(ncl * C);
      const int iters = 200;
      const double ms = timeit([&] { CK(cudaLaunchKernelEx(&lc, fn, C, iters, sink)); });
      const double bytes = (double)ncl * C * iters * 65536;
      printf("dsmbw C=%d clusters=%d: %.0f GB/s total, %.1f B/clk/SM at 1.9 GHz\n", C, ncl, bytes / (ms * 1e6),
             bytes / (ms * 1e-3) / (ncl * C) / 1.9e9);
      fflush(stdout);
    }
  }
  return 0;
}

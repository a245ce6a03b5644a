// lean.cu -- lean staged passes for the large power-of-two complex64 DFTs.
//
// Same algorithm as the generic staged pass (efft_kernels.cuh: the four-step
// form of the reference's scatter -> leaves -> merges, scatter.py:31-57,
// leaf_dft.py:93-125, recombine.py:144-260), specialised so that a tile costs
// as few issue slots and registers as possible:
//   * 512 threads x 16 complex64 elements (64 regs/thread -> 2 CTAs, 32 warps
//     per SM: enough warps in flight to hide HBM / L2 latency without any
//     explicit prefetch machinery);
//   * every global access is one 8-byte element per lane, 16 lanes covering
//     one 128-byte line (half-warp granularity), so the 16 points a thread
//     owns for its first radix stage come straight from HBM / L2 into
//     registers;
//   * exactly one shared-memory exchange per sub-stage (one STS + one LDS per
//     element, XOR-swizzled where the exchange also transposes);
//   * radix-16 / radix-8 register DFTs in paired-fp32 (FADD2/FFMA2) arithmetic;
//   * twiddles from per-CTA tables computed in fp64 (W_256, W_R^(i<256),
//     three 1024-entry levels of W_N) with short fp32 recurrences: no twiddle
//     array is read from HBM.
//
// Index maps (N = R1 R2, R = 256 RB per pass, j = ja + RB jb, k = kb + 256 ka,
// jb = s + 16 t, kb = kt + 16 ks, ja = p + 16 q, ka = kq + QB kp):
//   pass 1 (T1):  x[j2 + R2 j1] -> y[k1 + R1 j2] * W_N^(j2 k1); group = 16 j2
//   pass 2 (T0):  y[k1 + R1 j2] -> X[k1 + R1 k2] in place;      group = 16 k1
// Sub-stage A (per group: RB/2 tiles of 16 lanes x 256 jb x 2 ja):
//   16-point DFT over t, W_256^(s kt), exchange, 16-point DFT over s,
//   store to the group's L2 staging slot (T1: lanes become kt -- the transpose).
// Sub-stage B (RB/2 tiles of 16 lanes x RB ja x (512/RB) kb or j2):
//   W_R^(ja kb), QB-point DFT over q, W_RB^(p kq), exchange, 16-point DFT over
//   p, (T1: W_N^(j2 k1)), store to HBM.
#include "efft_kernels.cuh"
#include "lean.cuh"

#include <cstdlib>

namespace efft {
namespace lean {

constexpr int NT = 256;
constexpr int XB_ELEMS = 256 * 17;  // exchange buffer (4096 elements, T1 rows padded to 17)
using V = float2;

template <int S>
__device__ __forceinline__ constexpr int P(int k) {
  return dif_pos(S, k);
}

__device__ __forceinline__ V ld_hbm(const V* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return *reinterpret_cast<V*>(&r);
}
__device__ __forceinline__ V ld_l2(const V* p) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return *reinterpret_cast<V*>(&r);
}

// W_R^e, e < R = 256 RB: W_RB^(e >> 8) * W_R^(e & 255)
template <int RB>
__device__ __forceinline__ V w_pass(const V* w256, const V* wlo, int e) {
  return cmul(w256[(e >> 8) * (256 / RB)], wlo[e & 255]);
}
// W_N^e, e < N <= 2^30: three 10-bit levels
__device__ __forceinline__ V w_full(const V* t4, uint32_t e) {
  return cmul(cmul(__ldg(t4 + (e >> 20)), __ldg(t4 + 1024 + ((e >> 10) & 1023))), __ldg(t4 + 2048 + (e & 1023)));
}

// ---------------------------------------------------------------------------
// sub-stage A: one unit ja of one group (16 lanes x 256 jb).  The tile has
// landed in `buf` as [jb][lane] (TMA).
// ---------------------------------------------------------------------------
template <int RB, bool T1>
__device__ __forceinline__ void tile_a(const Args& a, int g, int ja, int slot, V* buf, const V* w256, bool& nf) {
  const int tid = threadIdx.x, lane = tid & 15, r = tid >> 4;
  V v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = buf[(r + 16 * t) * 16 + lane];  // jb = s + 16 t, s = r
  if (a.check_finite) {
#pragma unroll
    for (int t = 0; t < 16; ++t) nf |= !(isfinite(v[t].x) && isfinite(v[t].y));
  }
  if constexpr (T1) {
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = mul2(v[t], a.cin);
  }
  reg_dft<float, 16>(v);  // over t
  {
    const V* wp = w256;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      wp += r;
      v[P<16>(k)] = cmul(v[P<16>(k)], *wp);  // W_256^(s k)
    }
  }
  // the staging slot must have been released by B(g - nslots)
  if (tid == 0 && g >= a.nslots) {
    const int32_t* c = a.doneB + (g - a.nslots);
    long long n = 0;
    while (ld_acquire(c) < a.nt) {
      __nanosleep(32);
      if (++n == (1ll << 26)) {
        printf("EFFT lean STUCK (A) cta=%d g=%d\n", blockIdx.x, g);
        __trap();
      }
    }
  }
  __syncthreads();  // every stage-0 read of buf is done
  // exchange in buf.  T0: [kt][s][lane].  T1 (transpose lanes j2 -> kt):
  // [s][kt][j2], row pitch 17 so that both the write (lanes = j2) and the read
  // (lanes = kt) hit 16 distinct 8-byte bank pairs.
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if constexpr (T1)
      buf[r * 272 + k * 17 + lane] = v[P<16>(k)];
    else
      buf[k * 256 + r * 16 + lane] = v[P<16>(k)];
  }
  __syncthreads();
  // stage 1.  T0 thread (lane, kt = r);  T1 thread (kt = lane, j2l = r)
#pragma unroll
  for (int u = 0; u < 16; ++u) v[u] = T1 ? buf[u * 272 + lane * 17 + r] : buf[r * 256 + u * 16 + lane];
  reg_dft<float, 16>(v);  // over s -> ks
  V* sp = a.stg + (int64_t)slot * a.slot_elems;
  int base, step;
  if constexpr (T1) {  // staging [j2l][ja][ks][kt]
    base = (r * RB + ja) * 256 + lane;
    step = 16;
  } else {  // staging [kb][ja][lane], kb = kt + 16 ks
    base = (r * RB + ja) * 16 + lane;
    step = 16 * RB * 16;
  }
  const uint64_t keep = policy_evict_last();
#pragma unroll
  for (int ks = 0; ks < 16; ++ks) st_hint(sp + base + ks * step, v[P<16>(ks)], keep);
}

// ---------------------------------------------------------------------------
// sub-stage B: 16 lanes x RB ja x DB (kb or j2) of one group, landed in `buf`
// as [dl][ja][lane].
// ---------------------------------------------------------------------------
template <int RB, bool T1>
__device__ __forceinline__ void tile_b(const Args& a, int g, int task, V* buf, const V* w256, const V* wlo) {
  constexpr int QB = RB / 16, DB = 16 / QB;
  const int tid = threadIdx.x, lane = tid & 15, p = tid >> 4;
  V v[16];
#pragma unroll
  for (int dl = 0; dl < DB; ++dl)
#pragma unroll
    for (int q = 0; q < QB; ++q) v[dl * QB + q] = buf[(dl * RB + p + 16 * q) * 16 + lane];
  // W_R^(ja kb), ja = p + 16 q: exact base and step, recurrence over q
#pragma unroll
  for (int dl = 0; dl < DB; ++dl) {
    const int kb = T1 ? lane + 16 * (task & 15) : task * DB + dl;
    V w = w_pass<RB>(w256, wlo, p * kb);
    const V st = w_pass<RB>(w256, wlo, (16 * kb) & (256 * RB - 1));
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      v[dl * QB + q] = cmul(v[dl * QB + q], w);
      if (q + 1 < QB) w = cmul(w, st);
    }
  }
#pragma unroll
  for (int dl = 0; dl < DB; ++dl) reg_dft<float, QB>(v + dl * QB);
  // inner twiddle W_RB^(p kq)
  {
    const V* wp = w256;
#pragma unroll
    for (int k = 1; k < QB; ++k) {
      wp += p * (256 / RB);
      const V w = *wp;
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) v[dl * QB + P<QB>(k)] = cmul(v[dl * QB + P<QB>(k)], w);
    }
  }
  __syncthreads();  // every stage-0 read of buf is done
#pragma unroll
  for (int dl = 0; dl < DB; ++dl)
#pragma unroll
    for (int k = 0; k < QB; ++k) buf[((dl * QB + k) * 16 + p) * 16 + lane] = v[dl * QB + P<QB>(k)];
  __syncthreads();
  const int kq = p % QB, dl = p / QB;  // stage-1 thread (lane, dl, kq)
#pragma unroll
  for (int u = 0; u < 16; ++u) v[u] = buf[((dl * QB + kq) * 16 + u) * 16 + lane];
  reg_dft<float, 16>(v);  // over p -> kp
  const uint64_t pol = policy_evict_first();
  if constexpr (T1) {
    // y[k1 + R1 j2] = Y * W_N^(j2 k1), k1 = kb + 256 kq + 256 QB kp, kb = lane + 16 ks
    const int kb = lane + 16 * (task & 15);
    const int j2 = g * 16 + (task >> 4) * DB + dl;
    const uint32_t c = (uint32_t)(kb + 256 * kq);
    V w = w_full(a.t4, (uint32_t)((uint64_t)j2 * c));
    const V st = w_full(a.t4, (uint32_t)(((uint64_t)j2 * (256 * QB)) & (uint64_t)(a.N - 1)));
    V* op = a.dst + (int64_t)j2 * a.R + c;
#pragma unroll
    for (int kp = 0; kp < 16; ++kp) {
      st_hint(op + kp * (256 * QB), cmul(v[P<16>(kp)], w), pol);
      if (kp < 15) w = cmul(w, st);
    }
  } else {
    const int kb = task * DB + dl;
    V* op = a.dst + (int64_t)g * 16 + lane + a.LS * (int64_t)(kb + 256 * kq);
    const int64_t step = a.LS * (int64_t)(256 * QB);
#pragma unroll
    for (int kp = 0; kp < 16; ++kp) st_hint(op + kp * step, mul2(v[P<16>(kp)], a.cout), pol);
  }
}

// ---------------------------------------------------------------------------
// persistent pass kernel, static schedule: CTA c runs task positions c, c+G,
// c+2G, ... of the order A(0..lag-1), [B(g-lag) x nt, A(g) x nt] pairs, the
// tail of B.  Thread 0 keeps the tiles of the next NBUF-1 positions in flight
// (TMA into NBUF shared-memory buffers, one mbarrier each); a buffer is
// refilled right after the tile in it has been finished and released.
// Dependencies: B(g)'s copy is issued only after A(g) is complete; A(g)'s
// staging stores wait for the slot release by B(g - nslots).  Every
// dependency points to a position at least lag*2*nt - nt > NBUF*G earlier,
// a CTA finishes and releases its positions in increasing order, and it never
// waits while holding an unreleased finished tile, so the smallest unfinished
// position can always progress: deadlock-free.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void decode(const Args& a, int lnt, long long pos, int& isB, int& g, int& task) {
  const long long L = a.lag, nt = a.nt, G = a.ngroups;
  if (pos < L * nt) {
    isB = 0;
    g = (int)(pos >> lnt);
    task = (int)(pos & (nt - 1));
  } else if (pos < L * nt + (G - L) * 2 * nt) {
    const long long q = pos - L * nt;
    const long long i = L + (q >> (lnt + 1)), r = q & (2 * nt - 1);
    isB = r < nt;
    g = (int)(isB ? i - L : i);
    task = (int)(r & (nt - 1));
  } else {
    const long long q = pos - L * nt - (G - L) * 2 * nt;
    isB = 1;
    g = (int)(G - L + (q >> lnt));
    task = (int)(q & (nt - 1));
  }
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int RB, bool T1, int NBUF, int MINB>
__global__ void __launch_bounds__(NT, MINB) lean_pass(const __grid_constant__ Args a) {
  constexpr int DB = 256 / RB;
  extern __shared__ __align__(128) unsigned char smraw[];
  V* bufs = reinterpret_cast<V*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
  V* w256 = bufs + NBUF * XB_ELEMS;
  V* wlo = w256 + 256;
  __shared__ __align__(8) uint64_t full[NBUF];
  const int tid = threadIdx.x;
  for (int i = tid; i < 256; i += NT) {
    w256[i] = to_v(wroot(i, 256), 0.f);
    wlo[i] = to_v(wroot(i, a.R), 0.f);
  }
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lnt = __ffs(a.nt) - 1;
  const long long G = gridDim.x;
  // thread 0: issue the copy of the tile at `pos` into buffer b
  auto issue = [&](long long pos, int b) {
    if (pos >= a.total) return;
    int isB, g, task;
    decode(a, lnt, pos, isB, g, task);
    V* dst = bufs + b * XB_ELEMS;
    if (isB) {
      const int32_t* c = a.doneA + g;
      long long n = 0;
      while (ld_acquire(c) < a.nt) {
        __nanosleep(32);
        if (++n == (1ll << 26)) {
          printf("EFFT lean STUCK (B) cta=%d g=%d\n", blockIdx.x, g);
          __trap();
        }
      }
      fence_proxy_async();
      mbar_arrive_tx(&full[b], 4096 * sizeof(V));
      const int slot = g % a.nslots;
      const uint64_t pol = policy_evict_first();
      if constexpr (T1)
        tma_load_5d(dst, &a.tmB, 0, task & 15, 0, (task >> 4) * DB, slot, &full[b], pol);
      else
        bulk_g2s(dst, a.stg + (int64_t)slot * a.slot_elems + (int64_t)task * 4096, 4096 * sizeof(V), &full[b], pol);
    } else {
      mbar_arrive_tx(&full[b], 4096 * sizeof(V));
      tma_load_4d(dst, &a.tmA, 0, g, task, 0, &full[b], policy_evict_first());
    }
  };
  if (tid == 0)
    for (int k = 0; k < NBUF; ++k) issue(blockIdx.x + k * G, k);
  bool nf = false;
  for (int k = 0;; ++k) {
    const long long pos = blockIdx.x + k * G;
    if (pos >= a.total) break;
    int isB, g, task;
    decode(a, lnt, pos, isB, g, task);
    const int b = k % NBUF;
    V* buf = bufs + b * XB_ELEMS;
    mbar_wait(&full[b], (uint32_t)((k / NBUF) & 1));
    if (isB) {
      // drop the consumed staging lines from L2 (no write-back): the tile is in smem
      const V* sp = a.stg + (int64_t)(g % a.nslots) * a.slot_elems;
      const int dl = tid / RB, ja = tid % RB;
      if constexpr (T1)
        l2_discard(sp + ((((task >> 4) * DB + dl) * RB + ja) * 16 + (task & 15)) * 16);
      else
        l2_discard(sp + (int64_t)task * 4096 + tid * 16);
      tile_b<RB, T1>(a, g, task, buf, w256, wlo);
    } else {
      tile_a<RB, T1>(a, g, task, g % a.nslots, buf, w256, nf);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      red_release_add(isB ? a.doneB + g : a.doneA + g, 1);
      issue(pos + NBUF * G, b);
    }
  }
  if (__syncthreads_or(nf) && tid == 0) atomicOr(a.flag, 1);
}

// ---------------------------------------------------------------------------
// Register-fed variant (default): the tile's 16 points per thread are loaded
// straight into registers (4 CTAs x 256 threads per SM).  Synchronisation is
// kept off the critical path: thread 0 checks the next task's dependency with
// an acquire load issued next to its own tile loads (same latency), and the
// completion of tile k is released in the middle of tile k+1 (after its
// stage-0 work, when tile k's stores have long been acknowledged), so no warp
// waits on a fence round trip.
// ---------------------------------------------------------------------------
template <int RB, bool T1>
__device__ __forceinline__ void ra_tile_a_load(const Args& a, int g, int ja, V* v) {
  const int lane = threadIdx.x & 15, r = threadIdx.x >> 4;
  const uint64_t pol = policy_evict_first();
  const V* sp = a.src + (int64_t)g * 16 + lane + a.LS * (int64_t)(ja + RB * r);
  const int64_t step = a.LS * (int64_t)(RB * 16);
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = ld_hbm(sp + t * step, pol);
}

template <int RB, bool T1>
__device__ __forceinline__ void ra_tile_b_load(const Args& a, int task, int slot, V* v) {
  constexpr int QB = RB / 16, DB = 16 / QB;
  const int lane = threadIdx.x & 15, p = threadIdx.x >> 4;
  const V* sp = a.stg + (int64_t)slot * a.slot_elems;
  constexpr int QSTEP = T1 ? 16 * 16 * 16 : 16 * 16;
#pragma unroll
  for (int dl = 0; dl < DB; ++dl) {
    const int lb = T1 ? ((((task >> 4) * DB + dl) * RB + p) * 16 + (task & 15)) * 16 : ((task * DB + dl) * RB + p) * 16;
    const V* b = sp + lb + lane;
#pragma unroll
    for (int q = 0; q < QB; ++q) v[dl * QB + q] = ld_l2(b + q * QSTEP);
  }
}

// thread 0's synchronisation state
struct Sync {
  int32_t* pend;  // completion counter of the finished, not yet released tile
  __device__ __forceinline__ void flush() {
    if (pend != nullptr) {
      __threadfence();
      red_release_add(pend, 1);
      pend = nullptr;
    }
  }
  __device__ __forceinline__ void spin(const int32_t* c, int32_t need, int tag) {
    long long n = 0;
    while (ld_acquire(c) < need) {
      __nanosleep(32);
      if (++n == (1ll << 26)) {
        printf("EFFT lean STUCK (%d) cta=%d\n", tag, blockIdx.x);
        __trap();
      }
    }
  }
};

template <int RB, bool T1>
__global__ void __launch_bounds__(NT, 4) lean_reg(const __grid_constant__ Args a) {
  constexpr int QB = RB / 16, DB = 16 / QB;
  extern __shared__ __align__(128) unsigned char smraw[];
  V* xb = reinterpret_cast<V*>(smraw);
  V* w256 = xb + XB_ELEMS;
  V* wlo = w256 + 256;
  __shared__ int s_ready;
  const int tid = threadIdx.x, lane = tid & 15, r = tid >> 4;
  for (int i = tid; i < 256; i += NT) {
    w256[i] = to_v(wroot(i, 256), 0.f);
    wlo[i] = to_v(wroot(i, a.R), 0.f);
  }
  const int lnt = __ffs(a.nt) - 1;
  const long long G = gridDim.x;
  Sync sy{nullptr};
  // dependency counter (and its target) that must be complete before a task's
  // loads (B: its A tiles) -- A tasks depend only at store time
  auto dep_b = [&](long long pos, const int32_t*& c) -> bool {
    if (pos >= a.total) return false;
    int isB, g, task;
    decode(a, lnt, pos, isB, g, task);
    c = a.doneA + g;
    return isB;
  };
  // Dynamic schedule, claims two tasks ahead (the atomic's latency hides
  // behind a whole tile).  Claims of one CTA increase monotonically.
  __shared__ long long s_cur, s_nxt;
  if (tid == 0) {
    s_cur = (long long)atomicAdd(a.ctr, 1ull);
    s_nxt = (long long)atomicAdd(a.ctr, 1ull);
    const int32_t* c;
    s_ready = !dep_b(s_cur, c) || ld_acquire(c) >= a.nt;
  }
  __syncthreads();
  bool nf = false;
  for (;;) {
    const long long pos = s_cur;
    if (pos >= a.total) break;
    int isB, g, task;
    decode(a, lnt, pos, isB, g, task);
    const int slot = g % a.nslots;
    if (isB && !s_ready) {  // rare: the producers of this B tile were late
      if (tid == 0) {
        sy.flush();
        sy.spin(a.doneA + g, a.nt, 1);
      }
      __syncthreads();
    }
    V v[16];
    if (isB)
      ra_tile_b_load<RB, T1>(a, task, slot, v);
    else
      ra_tile_a_load<RB, T1>(a, g, task, v);
    // thread 0: claim the task after next, acquire-probe the next task's
    // producers and this A task's slot (latency hidden behind the tile loads)
    int32_t nxt_val = 0;
    const int32_t* nxt_c = nullptr;
    bool nxt_isB = false;
    int32_t slot_val = a.nt;
    long long claim2 = 0;
    if (tid == 0) {
      claim2 = (long long)atomicAdd(a.ctr, 1ull);
      nxt_isB = dep_b(s_nxt, nxt_c);
      if (nxt_isB) nxt_val = ld_acquire(nxt_c);
      if (!isB && g >= a.nslots) slot_val = ld_acquire(a.doneB + (g - a.nslots));
    }
    const bool compute = !(a.check_finite & 2);  // diagnostic: bit 1 skips the arithmetic
    if (isB) {
      // -------- sub-stage B, stage 0 --------
#pragma unroll
      for (int dl = 0; dl < DB && compute; ++dl) {
        const int kb = T1 ? lane + 16 * (task & 15) : task * DB + dl;
        V w = w_pass<RB>(w256, wlo, r * kb);
        const V st = w_pass<RB>(w256, wlo, (16 * kb) & (256 * RB - 1));
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          v[dl * QB + q] = cmul(v[dl * QB + q], w);
          if (q + 1 < QB) w = cmul(w, st);
        }
      }
#pragma unroll
      for (int dl = 0; dl < DB && compute; ++dl) reg_dft<float, QB>(v + dl * QB);
      if (compute) {
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < QB; ++k) {
          wp += r * (256 / RB);
          const V w = *wp;
#pragma unroll
          for (int dl = 0; dl < DB; ++dl) v[dl * QB + P<QB>(k)] = cmul(v[dl * QB + P<QB>(k)], w);
        }
      }
      {  // the consumed staging lines: lane i drops the line of its own load i
        const V* sp = a.stg + (int64_t)slot * a.slot_elems;
        const int dl = lane / QB, q = lane % QB;
        const int lb = T1 ? ((((task >> 4) * DB + dl) * RB + r) * 16 + (task & 15)) * 16 : ((task * DB + dl) * RB + r) * 16;
        l2_discard(sp + lb + q * (T1 ? 4096 : 256));
      }
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int k = 0; k < QB; ++k) xb[((dl * QB + k) * 16 + r) * 16 + lane] = v[dl * QB + P<QB>(k)];
    } else {
      // -------- sub-stage A, stage 0 --------
      if (a.check_finite & 1) {
#pragma unroll
        for (int t = 0; t < 16; ++t) nf |= !(isfinite(v[t].x) && isfinite(v[t].y));
      }
      if constexpr (T1) {
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = mul2(v[t], a.cin);
      }
      if (compute) {
        reg_dft<float, 16>(v);
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < 16; ++k) {
          wp += r;
          v[P<16>(k)] = cmul(v[P<16>(k)], *wp);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if constexpr (T1)
          xb[r * 272 + k * 17 + lane] = v[P<16>(k)];
        else
          xb[k * 256 + r * 16 + lane] = v[P<16>(k)];
      }
      if (tid == 0 && slot_val < a.nt) {  // rare: the slot is still being read
        sy.flush();
        sy.spin(a.doneB + (g - a.nslots), a.nt, 2);
      }
    }
    if (tid == 0) sy.flush();  // release the previous tile (its stores are long done)
    __syncthreads();
    if (isB) {
      const int kq = r % QB, dl = r / QB;
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = xb[((dl * QB + kq) * 16 + u) * 16 + lane];
      if (compute) reg_dft<float, 16>(v);
      const uint64_t pol = policy_evict_first();
      if constexpr (T1) {
        const int kb = lane + 16 * (task & 15);
        const int j2 = g * 16 + (task >> 4) * DB + dl;
        const uint32_t c = (uint32_t)(kb + 256 * kq);
        V w = w_full(a.t4, (uint32_t)((uint64_t)j2 * c));
        const V st = w_full(a.t4, (uint32_t)(((uint64_t)j2 * (256 * QB)) & (uint64_t)(a.N - 1)));
        V* op = a.dst + (int64_t)j2 * a.R + c;
#pragma unroll
        for (int kp = 0; kp < 16; ++kp) {
          st_hint(op + kp * (256 * QB), cmul(v[P<16>(kp)], w), pol);
          if (kp < 15) w = cmul(w, st);
        }
      } else {
        const int kb = task * DB + dl;
        V* op = a.dst + (int64_t)g * 16 + lane + a.LS * (int64_t)(kb + 256 * kq);
        const int64_t step = a.LS * (int64_t)(256 * QB);
#pragma unroll
        for (int kp = 0; kp < 16; ++kp) st_hint(op + kp * step, mul2(v[P<16>(kp)], a.cout), pol);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = T1 ? xb[u * 272 + lane * 17 + r] : xb[r * 256 + u * 16 + lane];
      if (compute) reg_dft<float, 16>(v);
      V* sp = a.stg + (int64_t)slot * a.slot_elems;
      const int base = T1 ? (r * RB + task) * 256 + lane : (r * RB + task) * 16 + lane;
      const int step = T1 ? 16 : 16 * RB * 16;
      const uint64_t keep = policy_evict_last();
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) st_hint(sp + base + ks * step, v[P<16>(ks)], keep);
    }
    if (tid == 0) {
      s_ready = !nxt_isB || nxt_val >= a.nt;
      sy.pend = isB ? a.doneB + g : a.doneA + g;
      s_cur = s_nxt;
      s_nxt = claim2;
    }
    __syncthreads();
  }
  if (tid == 0) sy.flush();
  if (__syncthreads_or(nf) && tid == 0) atomicOr(a.flag, 1);
}

__global__ void tables_kernel(float2* t4, int64_t n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3072) return;
  const int lvl = i >> 10, j = i & 1023;
  const int64_t ex = ((int64_t)j << (10 * (2 - lvl))) & (n - 1);
  t4[i] = to_v(wroot(ex, n), 0.f);
}

void build_tables(float2* t4, int64_t n, cudaStream_t s) { tables_kernel<<<12, 256, 0, s>>>(t4, n); }

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// kernel configurations: {buffers per CTA, CTAs per SM}
struct Cfg {
  int nbuf, minb;
};
static const Cfg kCfgs[] = {{0, 4}, {2, 3}, {3, 2}, {4, 1}};  // cfg 0: register-fed (lean_reg)

template <int RB, bool T1>
static void* fn_of(int cfg) {
  switch (cfg) {
    case 1: return (void*)lean_pass<RB, T1, 2, 3>;
    case 2: return (void*)lean_pass<RB, T1, 3, 2>;
    case 3: return (void*)lean_pass<RB, T1, 4, 1>;
    default: return (void*)lean_reg<RB, T1>;
  }
}

static void* pick(int rb, bool t1, int cfg) {
  switch (rb) {
    case 32: return t1 ? fn_of<32, true>(cfg) : fn_of<32, false>(cfg);
    case 64: return t1 ? fn_of<64, true>(cfg) : fn_of<64, false>(cfg);
    case 128: return t1 ? fn_of<128, true>(cfg) : fn_of<128, false>(cfg);
    case 256: return t1 ? fn_of<256, true>(cfg) : fn_of<256, false>(cfg);
    default: return nullptr;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// A tiles: src viewed as [lane (16), group (LS/16), ja (RB), jb (256)]
bool encode_src(Pass& q, const void* src) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const Args& a = q.a;
  cuuint64_t dims[4] = {16, (cuuint64_t)(a.LS / 16), (cuuint64_t)q.rb, 256};
  cuuint64_t strides[3] = {128, (cuuint64_t)(a.LS * 8), (cuuint64_t)(a.LS * q.rb * 8)};
  cuuint32_t box[4] = {16, 1, 1, 256};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&q.a.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(src), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  q.tmA_src = src;
  return true;
}

// T1 B tiles: the ring viewed as [kt (16), ks (16), ja (RB), j2l (16), slot]
bool encode_stg(Pass& q, void* stg, int nslots_total) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const int rb = q.rb;
  cuuint64_t dims[5] = {16, 16, (cuuint64_t)rb, 16, (cuuint64_t)nslots_total};
  cuuint64_t strides[4] = {128, 16 * 128, (cuuint64_t)rb * 16 * 128, (cuuint64_t)q.a.slot_elems * 8};
  cuuint32_t box[5] = {16, 1, (cuuint32_t)rb, (cuuint32_t)(256 / rb), 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&q.a.tmB, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, stg, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool plan(int64_t n, int inverse, bool scale_inverse, bool check_finite, int num_sms, Pass p[2],
          int64_t* staging_elems, int* err_cuda) {
  *err_cuda = 0;
  if (n <= 0 || (n & (n - 1))) return false;
  int L = 0;
  while ((int64_t(1) << L) < n) ++L;
  if (L < 26 || L > 30) return false;
  const int L1 = (L + 1) / 2, L2 = L - L1;
  if (L1 < 13 || L1 > 16 || L2 < 13 || L2 > 16) return false;
  const int64_t R1 = int64_t(1) << L1, R2 = int64_t(1) << L2;
  int64_t stg = 0;
  for (int i = 0; i < 2; ++i) {
    Pass& q = p[i];
    const bool t1 = i == 0;
    const int64_t R = t1 ? R1 : R2;
    q.rb = (int)(R / 256);
    int cfg = 0;
    if (const char* ev = getenv("EFFT_LEAN_CFG")) cfg = atoi(ev);
    if (cfg < 0 || cfg > 3) cfg = 0;
    const int nbuf = kCfgs[cfg].nbuf;
    q.fn = reinterpret_cast<void (*)(Args)>(pick(q.rb, t1, cfg));
    if (!q.fn) return false;
    q.nt = NT;
    q.smem = (int)(((nbuf ? nbuf : 1) * XB_ELEMS + 256 + 256) * sizeof(V)) + 128;
    Args& a = q.a;
    a = Args{};
    a.R = R;
    a.N = n;
    a.LS = t1 ? R2 : R1;
    a.ngroups = (int32_t)((t1 ? R2 : R1) / 16);
    a.nt = q.rb;
    a.slot_elems = 16 * R;
    a.total = (int64_t)a.ngroups * 2 * a.nt;
    a.cin = make_float2(1.f, t1 && inverse ? -1.f : 1.f);
    const float sc = (!t1 && inverse && scale_inverse) ? (float)(1.0 / (double)n) : 1.f;
    a.cout = make_float2(sc, (!t1 && inverse) ? -sc : sc);
    a.check_finite = t1 && check_finite;
    if (const char* ev = getenv("EFFT_LEAN_DIAG")) a.check_finite |= atoi(ev) << 1;
    if (cudaFuncSetAttribute((const void*)q.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, q.smem) != cudaSuccess) {
      *err_cuda = 1;
      return false;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)q.fn, NT, q.smem) != cudaSuccess || occ < 1) {
      *err_cuda = 1;
      return false;
    }
    q.grid = occ * num_sms;
    const int64_t per = 2 * (int64_t)a.nt;
    // positions in flight span about (NBUF + 1) * grid: B(g) must come at least that far after A(g)
    const int64_t window = ((nbuf + 4) * (int64_t)q.grid + per - 1) / per;
    int64_t lag = window + 1;
    if (const char* ev = getenv("EFFT_LEAN_LAG")) lag = atoi(ev);
    int64_t slots = lag + window + 2;
    if (const char* ev = getenv("EFFT_LEAN_SLOTS")) slots = atoi(ev);
    if (lag < 1) lag = 1;
    if (lag > a.ngroups) lag = a.ngroups;
    if (slots < lag + 1) slots = lag + 1;
    if (slots > a.ngroups) slots = a.ngroups;
    a.lag = (int32_t)lag;
    a.nslots = (int32_t)slots;
    q.counter_ints = 2 + 2 * (int64_t)a.ngroups;
    if (slots * a.slot_elems > stg) stg = slots * a.slot_elems;
  }
  *staging_elems = stg;
  return true;
}

}  // namespace lean
}  // namespace efft

// lean.cu -- lean staged passes for the large DFTs: complex64 and complex128,
// N = 2^k (2^26 <= N <= 2^32; complex64 from 2^24) and N = M * 2^k, M in
// {3, 5, 7} (about 2^24 .. 2^31 points).
//
// Same algorithm as the generic staged pass (efft_kernels.cuh: the four-step
// form of the reference's scatter -> leaves -> merges, scatter.py:31-57,
// leaf_dft.py:93-125, recombine.py:144-260), specialised so that a tile costs
// as few issue slots, registers and memory requests as possible:
//   * a tile is F columns (F = one 128-byte line: 16 c64 / 8 c128) x 256
//     points (32 KB), 4 CTAs per SM;
//   * lean_pass (complex128, and the 3 * 2^k pass): one element per lane, 16
//     points per thread, 16F threads;  lean_pair (complex64): two adjacent
//     columns per thread, 32 points per thread, 128 threads, so every HBM / L2
//     access is 16 bytes (8 lanes per line);
//   * the points a thread owns for its first radix stage come straight from
//     HBM / L2 into registers; exactly one shared-memory exchange per
//     sub-stage; the transposing exchange uses padded rows so both sides are
//     bank-conflict free;
//   * radix-16 / 12 / QB register DFTs (paired-fp32 FADD2/FFMA2 for c64);
//   * twiddles: W_256 and W_R^(i<256) in shared memory (built per CTA in fp64,
//     rounded once); the pass-1 four-step twiddle W_N^(j2 k1) from the exact
//     integer exponent -- fp64 sincospi base and step, fp64 recurrence, one
//     rounding per use.  No global twiddle table is read.
//
// Index maps (N = R1 R2, R = RA RB per pass, j = ja + RB jb, k = kb + RA ka,
// jb = s + A1 t, kb = kt + A0 ks (RA = A0 A1: 16 x 16, or 12 / 10 / 14 x 16
// for the factor 3 / 5 / 7), ja = p + 16 q, ka = kq + QB kp, QB = RB/16):
//   pass 1 (T1):  x[j2 + R2 j1] -> y[k1 + R1 j2] * W_N^(j2 k1); group = F j2
//   pass 2 (T0):  y[k1 + R1 j2] -> X[k1 + R1 k2] in place;      group = F k1
// Sub-stage A (per group: RB tiles of F lanes x RA jb, one ja each):
//   A0-point DFT over t, W_RA^(s kt), exchange, A1-point DFT over s, store to
//   the group's L2 staging slot (T1: lanes become kt -- the j2 <-> k1 transpose).
// Sub-stage B (per group: RA RB / 256 tiles of F lanes x RB ja x DB = 16/QB kb or j2):
//   W_R^(ja kb), QB-point DFTs over q, W_RB^(p kq), exchange, 16-point DFT over
//   p, (T1: W_N^(j2 k1)), store to HBM.
//
// Scheduling: one persistent kernel per pass.  Tasks are claimed from a
// counter in the order A(0..lag-1), [B(g-lag), A(g)] blocks, the tail of B;
// B(g) needs A(g) complete, A(g)'s staging stores need the slot released by
// B(g - nslots).  Every dependency points to an earlier position and a CTA's
// claims increase, so the smallest unfinished task can always run
// (deadlock-free; a CTA never blocks while holding an unreleased finished
// tile).  Thread 0 keeps synchronisation off the critical path (Sched below):
// claims run two tasks ahead, the next task's producers are probed with
// relaxed loads, and ONE fence.acq_rel per tile, issued right after the tile
// loads, releases the previous tile and completes those acquires.
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "efft_kernels.cuh"
#include "lean.cuh"

namespace efft {
namespace lean {

template <typename R>
struct LT {
  using V = typename CT<R>::V;
  static constexpr int F = 128 / (int)sizeof(V);  // lanes per 128-byte line
  static constexpr int NT = 16 * F;               // threads per tile
  static constexpr int TILE = 256 * F;            // elements per tile (32 KB)
  static constexpr int PITCH = F + 1;             // row pitch of the transposing exchange
  static constexpr int XB = 256 * PITCH;          // exchange buffer elements
};

template <int S>
__device__ __forceinline__ constexpr int P(int k) {
  return dif_pos_t<S>(k);
}

// one element per lane: HBM stream (L1 bypass, L2 evict-first hint)
template <typename V>
__device__ __forceinline__ V ld_hbm(const V* p, uint64_t pol) {
  if constexpr (sizeof(V) == 8) {
    uint2 r;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(pol));
    return *reinterpret_cast<V*>(&r);
  } else {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return *reinterpret_cast<V*>(&r);
  }
}

__device__ __forceinline__ float2 cscale(float2 v, float2 c) { return mul2(v, c); }
__device__ __forceinline__ double2 cscale(double2 v, double2 c) { return make_double2(v.x * c.x, v.y * c.y); }
__device__ __forceinline__ float2 cvt(double2 c, float) { return make_float2((float)c.x, (float)c.y); }
__device__ __forceinline__ double2 cvt(double2 c, double) { return c; }

// Pass-1 output offset of (local column j2, k1): the transposed layout
// y[k1 + R j2], or, for the sharded transform's NCCL path (a.obl = log2 L1 >
// 0), blocked by destination rank: [k1 / L1][j2][k1 % L1] (the all-to-all
// send buffer, no pack pass).  k1 and k1 + 1 always share a block.
__device__ __forceinline__ int64_t t1_out(const Args& a, int j2, uint32_t k1) {
  if (a.obl == 0) return (int64_t)j2 * a.R + k1;
  const uint32_t bl = 1u << a.obl;
  return ((int64_t)(k1 >> a.obl) * a.LS + j2) * bl + (k1 & (bl - 1));
}

// Position -> (sub-stage, group, task) of the claim order above (thread 0 only).
__device__ __forceinline__ void decode(const Args& a, uint32_t pos, int& isB, int& g, int& task) {
  // Super-groups of W = a.wg adjacent column groups: the order is the
  // group-level order of the super-groups with each block's tasks interleaved
  // over its W groups, so W adjacent 128-byte segments of every row are read
  // (and, in B, written) at about the same time -- DRAM page locality.
  // lag counts super-groups; dependencies stay per group.
  const uint32_t W = a.wg, L = a.lag, na = a.ntA * W, nb = a.ntB * W, per = na + nb, G = a.ngroups / W;
  uint32_t sg, t;
  if (pos < L * na) {
    isB = 0;
    sg = pos / na;
    t = pos % na;
  } else if (pos < L * na + (G - L) * per) {
    const uint32_t q = pos - L * na;
    const uint32_t i = L + q / per, r = q % per;
    isB = r < nb;
    sg = isB ? i - L : i;
    t = isB ? r : r - nb;
  } else {
    const uint32_t q = pos - L * na - (G - L) * per;
    isB = 1;
    sg = G - L + q / nb;
    t = q % nb;
  }
  g = (int)(sg * W + t % W);
  task = (int)(t / W);
}

// thread 0's synchronisation state
struct Sync {
  int32_t* pend;  // completion counter of the finished, not yet released tile
  // release pattern: fence.acq_rel then a relaxed add.  The same fence also
  // completes the acquire of every relaxed probe thread 0 issued before it.
  __device__ __forceinline__ void fence_release() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (pend != nullptr) {
      asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(pend) : "memory");
      pend = nullptr;
    }
  }
  __device__ __forceinline__ void flush() {
    if (pend != nullptr) fence_release();
  }
  __device__ __forceinline__ void spin(const int32_t* c, int32_t need, int tag) {
    long long n = 0;
    while (ld_acquire(c) < need) {
      __nanosleep(32);
      if (++n == (1ll << 27)) {
        printf("EFFT lean pass stuck (%d) cta=%d\n", tag, blockIdx.x);
        __trap();
      }
    }
  }
};

__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// B tile of the transposing pass: task -> (ks, h, jblk); kt = h F + lane, ks < S
template <int F, int S>
__device__ __forceinline__ void t1_task(int task, int& ks, int& h, int& jblk) {
  ks = task % S;
  h = (task / S) % (16 / F);
  jblk = (task / S) / (16 / F);
}

// staging element offset of a B tile's load (dl, q) for this thread
template <typename R, int RA, int RB, bool T1>
__device__ __forceinline__ int b_line(int task, int dl, int p, int q, int lane) {
  constexpr int F = LT<R>::F, QB = RB / 16, DB = 16 / QB, S = RA / 16;
  const int ja = p + 16 * q;
  if constexpr (T1) {
    int ks, h, jblk;
    t1_task<F, S>(task, ks, h, jblk);
    return (((jblk * DB + dl) * RB + ja) * S + ks) * 16 + h * F + lane;
  } else {
    return ((task * DB + dl) * RB + ja) * F + lane;
  }
}

// Per-CTA task scheduling shared by the tile kernels (see the header comment):
// dynamic claims two ahead, decoded once by thread 0 into shared memory;
// relaxed probes of the next task's producers at the loop top; one fence per
// tile right after the tile loads (release of tile k-1, acquire of the probes).
struct SchedShared {
  int ready, isB[2], g[2], task[2];
  long long pos[2];
};

struct Sched {
  SchedShared* sh;
  int cb = 0;         // slot of the current task (the other holds the next)
  Sync sy{nullptr};   // thread 0
  int32_t nxt_val = 0, slot_val = 0;
  long long claim2 = 0;

  __device__ __forceinline__ void publish(const Args& a, int b, long long pos) {  // thread 0
    sh->pos[b] = pos;
    if (pos < a.total) {
      int isB, g, task;
      decode(a, (uint32_t)pos, isB, g, task);
      sh->isB[b] = isB;
      sh->g[b] = g;
      sh->task[b] = task;
    }
  }
  __device__ __forceinline__ void init(const Args& a) {  // all threads
    if (threadIdx.x == 0) {
      publish(a, 0, (long long)atomicAdd(a.ctr, 1ull));
      publish(a, 1, (long long)atomicAdd(a.ctr, 1ull));
      sh->ready = sh->pos[0] >= a.total || !sh->isB[0] || ld_acquire(a.doneA + sh->g[0]) >= a.ntA;
    }
    __syncthreads();
  }
  // loop top (all threads): the current task, or false when the pass is done.
  // Thread 0 also claims the task after next and probes (relaxed) the next
  // task's producers and this A task's staging slot; the fence in
  // after_loads() completes those acquires before anything depends on them.
  __device__ __forceinline__ bool next(const Args& a, int& isB, int& g, int& task) {
    if (sh->pos[cb] >= a.total) return false;
    isB = sh->isB[cb];
    g = sh->g[cb];
    task = sh->task[cb];
    if (isB && !sh->ready) {  // rare: the producers of this B tile were late
      if (threadIdx.x == 0) {
        sy.flush();
        sy.spin(a.doneA + g, a.ntA, 1);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      claim2 = (long long)atomicAdd(a.ctr, 1ull);
      const int nb = cb ^ 1;
      nxt_val = 0;
      slot_val = a.ntB;
      if (sh->pos[nb] < a.total && sh->isB[nb]) nxt_val = ld_relaxed(a.doneA + sh->g[nb]);
      if (!isB && g >= a.nslots) slot_val = ld_relaxed(a.doneB + (g - a.nslots));
    }
    return true;
  }
  // thread 0, right after issuing the tile loads: one fence (acquire of the
  // probes, release of the previous tile).  Warp 0 waits for its loads here
  // anyway, so the fence costs no extra time on the critical path.
  __device__ __forceinline__ void after_loads(const Args&, int, int) {
    if (threadIdx.x == 0) sy.fence_release();
  }
  // thread 0, before the exchange barrier: this A tile may store once its
  // staging slot is free (rarely not yet)
  __device__ __forceinline__ void before_exchange(const Args& a, int g) {
    if (threadIdx.x == 0 && slot_val < a.ntB) sy.spin(a.doneB + (g - a.nslots), a.ntB, 2);
  }
  __device__ __forceinline__ void end(const Args& a, int isB, int g) {  // all threads
    if (threadIdx.x == 0) {
      const int nb = cb ^ 1;
      sh->ready = sh->pos[nb] >= a.total || !sh->isB[nb] || nxt_val >= a.ntA;
      sy.pend = isB ? a.doneB + g : a.doneA + g;
      publish(a, cb, claim2);  // the current slot now holds the task after next
    }
    cb ^= 1;
    __syncthreads();
  }
  __device__ __forceinline__ void finish(const Args& a, bool nf) {
    if (threadIdx.x == 0) sy.flush();
    if (__syncthreads_or(nf) && threadIdx.x == 0) atomicOr(a.flag, 1);
  }
};

// Generic tile kernel: one element per lane.  A tiles: RA = 16 S points
// (S = 16, or 12 for the 3 * 2^k family); B tiles: RB = 16 QB points.
template <typename R, int RA, int RB, bool T1, int MINB>
__global__ void __launch_bounds__(LT<R>::NT, MINB) lean_pass(const __grid_constant__ Args a) {
  using V = typename LT<R>::V;
  constexpr int F = LT<R>::F, NT = LT<R>::NT, PITCH = LT<R>::PITCH;
  constexpr int S = RA / 16, QB = RB / 16, DB = 16 / QB;
  // A tile: jb = s + A1 t (s < A1 rows of threads, t < A0), stage 0 = A0-point
  // DFT over t, stage 1 = A1-point DFT over s, kb = kt + A0 ks.  RA = 192 runs
  // 12 x 16 in the in-place pass (every thread row loads) and 16 x 12 in the
  // transposing one (its output lines need 16 consecutive kt).
  constexpr int A0 = (RA == 256 || T1) ? 16 : RA / 16, A1 = RA / A0;
  extern __shared__ __align__(128) unsigned char smraw[];
  V* xb = reinterpret_cast<V*>(smraw);
  constexpr int XBN = T1 ? LT<R>::XB : 256 * LT<R>::F;  // the plain exchange needs no padding
  V* w256 = xb + XBN;        // W_256^i      (B inner twiddle, W_RB = W_256^(256/RB))
  V* wlo = w256 + 256;       // W_R^i, i < 256
  // W_(R/256)^i, i < R/256 and W_RA^i, i < RA (A inner twiddle): own tables
  // only when RA = 192; for RA = 256 both are strided views of W_256
  V* whi = RA == 256 ? w256 : wlo + 256;
  V* wa = RA == 256 ? w256 : wlo + 256 + RA;
  constexpr int HS = RA == 256 ? 256 / RB : 1;  // stride of whi
  // T1 B tiles: the tile's four-step twiddle factors, built once per tile in fp64 (below)
  // (complex128 only: the complex64 instantiation of this kernel is a fallback behind lean_pair
  // and would spill with the extra addressing)
  constexpr bool TWT = T1 && sizeof(R) == 8;
  __shared__ double2 twc[TWT ? DB * F : 1], twq[TWT ? 16 : 1], tws[TWT ? DB : 1];
  __shared__ SchedShared shs;
  const int tid = threadIdx.x, lane = tid % F, r = tid / F;
  // kernel parameters stay in the constant bank (read at use, no registers held)
#define SRC reinterpret_cast<const V*>(a.src)
#define DST reinterpret_cast<V*>(a.dst)
#define STG reinterpret_cast<V*>(a.stg)
  for (int i = tid; i < 256; i += NT) {
    w256[i] = to_v(wroot(i, 256), R());
    wlo[i] = to_v(wroot(i, a.R), R());
    if constexpr (RA != 256) {
      if (i < RA) {  // R / 256 = RA RB / 256 <= RA and RA entries
        whi[i] = to_v(wroot(i, a.R / 256), R());
        wa[i] = to_v(wroot(i, RA), R());
      }
    }
  }
  Sched sc{&shs};
  sc.init(a);
  bool nf = false;
  int isB, g, task;
  while (sc.next(a, isB, g, task)) {
    V* sp = STG + (int64_t)(g % a.nslots) * a.slot_elems;
    V v[16];
    if (isB) {
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int q = 0; q < QB; ++q) v[dl * QB + q] = ld_staging(sp + b_line<R, RA, RB, T1>(task, dl, r, q, lane));
    } else if (r < A1) {  // A: jb = s + A1 t with s = r
      const uint64_t pol = policy_evict_first();
      const V* p0 = SRC + (int64_t)g * F + lane + a.LS * (int64_t)(task + RB * r);
      const int64_t step = a.LS * (int64_t)(RB * A1);
#pragma unroll
      for (int t = 0; t < A0; ++t) v[t] = ld_hbm(p0 + t * step, pol);
    }
    sc.after_loads(a, isB, g);
    if (isB) {
      // ---- sub-stage B, stage 0: W_R^(ja kb) (exact base and step, recurrence over q)
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        int kb;
        if constexpr (T1) {
          int ks, h, jblk;
          t1_task<F, S>(task, ks, h, jblk);
          kb = h * F + lane + 16 * ks;
        } else {
          kb = task * DB + dl;
        }
        const int e0 = r * kb, es = 16 * kb;  // < R
        V w = cmul(whi[(e0 >> 8) * HS], wlo[e0 & 255]);
        const V st = cmul(whi[(es >> 8) * HS], wlo[es & 255]);
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          v[dl * QB + q] = cmul(v[dl * QB + q], w);
          if (q + 1 < QB) w = cmul(w, st);
        }
      }
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) reg_dft<R, QB>(v + dl * QB);
      {  // W_RB^(p kq)
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < QB; ++k) {
          wp += r * (256 / RB);
          const V w = *wp;
#pragma unroll
          for (int dl = 0; dl < DB; ++dl) v[dl * QB + P<QB>(k)] = cmul(v[dl * QB + P<QB>(k)], w);
        }
      }
      if constexpr (TWT) {
        // W_N^(j2 k1), k1 = c + RA QB kp, c = (h F + lane + 16 ks) + RA kq, from exact integer
        // exponents in fp64, factored so that a tile needs DB (F + QB + 1) sincospi instead of
        // two per thread: twc[dl][lane] = W_N^(j2 (h F + lane + 16 ks)), twq[dl][kq] = W_N^(j2 RA kq),
        // tws[dl] = W_N^(j2 RA QB) (the recurrence step)
        int ks, h, jblk;
        t1_task<F, S>(task, ks, h, jblk);
        const uint64_t N = (uint64_t)a.N;
        for (int i = tid; i < DB * F + 16 + DB; i += NT) {
          int dl2, kind, idx;
          if (i < DB * F) {
            kind = 0, dl2 = i / F, idx = i % F;
          } else if (i < DB * F + 16) {
            kind = 1, dl2 = (i - DB * F) / QB, idx = (i - DB * F) % QB;
          } else {
            kind = 2, dl2 = i - DB * F - 16, idx = 0;
          }
          const uint64_t jg = (uint64_t)(a.j2off + g * F + jblk * DB + dl2);  // global column
          const uint64_t m = kind == 0 ? (uint64_t)(h * F + idx + 16 * ks) : kind == 1 ? (uint64_t)(RA * idx)
                                                                                       : (uint64_t)(RA * QB);
          const double2 w = wroot((int64_t)((jg * m) % N), a.N);
          if (kind == 0) twc[i] = w;
          else if (kind == 1) twq[i - DB * F] = w;
          else tws[dl2] = w;
        }
      }
      // the consumed staging lines leave L2 without write-back: F lanes share
      // a line, lane i drops the lines of its loads i, i + F, ...
#pragma unroll
      for (int i = lane; i < 16; i += F) l2_discard(sp + b_line<R, RA, RB, T1>(task, i / QB, r, i % QB, 0));
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int k = 0; k < QB; ++k) xb[((dl * QB + k) * 16 + r) * F + lane] = v[dl * QB + P<QB>(k)];
    } else if (r < A1) {
      // ---- sub-stage A, stage 0: A0-point DFT over t, W_RA^(s kt)
      if (a.check_finite) {
#pragma unroll
        for (int t = 0; t < A0; ++t) nf |= !(isfinite(v[t].x) && isfinite(v[t].y));
      }
      if constexpr (T1) {
        if (a.cin.y != 1.0) {  // inverse: conjugate the input (forward: identity)
#pragma unroll
          for (int t = 0; t < A0; ++t) v[t] = cscale(v[t], cvt(a.cin, R()));
        }
      }
      reg_dft<R, A0>(v);
      {
        const V* wp = wa;
#pragma unroll
        for (int k = 1; k < A0; ++k) {
          wp += r;
          v[P<A0>(k)] = cmul(v[P<A0>(k)], *wp);
        }
      }
#pragma unroll
      for (int k = 0; k < A0; ++k) {
        if constexpr (T1)
          xb[(r * 16 + k) * PITCH + lane] = v[P<A0>(k)];  // [s][kt][j2l]
        else
          xb[(k * A1 + r) * F + lane] = v[P<A0>(k)];  // [kt][s][lane]
      }
    }
    sc.before_exchange(a, g);
    __syncthreads();
    if (isB) {
      // ---- sub-stage B, stage 1: 16-point DFT over p; stage-1 thread (lane, dl, kq)
      const int kq = r % QB, dl = r / QB;
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = xb[((dl * QB + kq) * 16 + u) * F + lane];
      reg_dft<R, 16>(v);
      const uint64_t pol = policy_evict_first();
      if constexpr (T1) {
        // y[k1 + R1 j2] = Y W_N^(j2 k1), k1 = kt + 16 ks + RA kq + RA QB kp
        int ks, h, jblk;
        t1_task<F, S>(task, ks, h, jblk);
        const int j2 = g * F + jblk * DB + dl;
        const uint32_t c = (uint32_t)(h * F + lane + 16 * ks + RA * kq);
        // W_N^(j2 k1) from the exact integer exponent: fp64 base and step
        // (sincospi), fp64 recurrence, one rounding per use (north star c)
        double2 w, st;
        if constexpr (TWT) {
          w = cmul(twc[dl * F + lane], twq[dl * QB + kq]);
          st = tws[dl];
        } else {
          const uint64_t jg = (uint64_t)(a.j2off + j2);  // global column (sharded: rank offset)
          w = wroot((int64_t)((jg * c) % (uint64_t)a.N), a.N);
          st = wroot((int64_t)((jg * (RA * QB)) % (uint64_t)a.N), a.N);
        }
        V* op = DST + (int64_t)j2 * a.R + c;
#pragma unroll
        for (int kp = 0; kp < 16; ++kp) {
          V* dp = a.obl == 0 ? op + kp * (RA * QB) : DST + t1_out(a, j2, c + kp * (RA * QB));
          st_hint(dp, cmul(v[P<16>(kp)], to_v(w, R())), pol);
          if (kp < 15) w = cmul(w, st);
        }
      } else {
        const int kb = task * DB + dl;
        V* op = DST + (int64_t)g * F + lane + a.LS * (int64_t)(kb + RA * kq);
        const int64_t step = a.LS * (int64_t)(RA * QB);
        if (RA == 256 && a.cout.x == 1.0 && a.cout.y == 1.0) {  // forward: no conjugation, no scale
          // (the odd-factor tiles keep the multiply: a second copy of the stores would spill)
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) st_hint(op + kp * step, v[P<16>(kp)], pol);
        } else {
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) st_hint(op + kp * step, cscale(v[P<16>(kp)], cvt(a.cout, R())), pol);
        }
      }
    } else if (T1 || r < A0) {
      // ---- sub-stage A, stage 1: A1-point DFT over s -> ks, store to the ring
      // T0 thread (lane, kt = r): ring [kb][ja][lane], kb = kt + A0 ks
      // T1 thread (kt = tid % 16, j2l = tid / 16): ring [j2l][ja][ks][kt]
      const int kt = T1 ? tid % 16 : r, j2l = tid / 16;
#pragma unroll
      for (int u = 0; u < A1; ++u) v[u] = T1 ? xb[(u * 16 + kt) * PITCH + j2l] : xb[(kt * A1 + u) * F + lane];
      reg_dft<R, A1>(v);
      const int base = T1 ? (j2l * RB + task) * (16 * A1) + kt : (kt * RB + task) * F + lane;
      const int step = T1 ? 16 : A0 * RB * F;
      const uint64_t keep = policy_evict_last();
#pragma unroll
      for (int ks = 0; ks < A1; ++ks) st_hint(sp + base + ks * step, v[P<A1>(ks)], keep);
    }
    sc.end(a, isB, g);
  }
  sc.finish(a, nf);
#undef SRC
#undef DST
#undef STG
}

// Paired-column complex64 tile kernel (the default for complex64, RA = 256):
// each thread owns two adjacent columns, so every global and most shared
// accesses are 16 bytes (8 lanes per 128-byte line: half the memory requests
// of the one-element-per-lane kernel -- the request rate, not the bytes in
// flight, bounds a 128-byte-line gather on B200).  32 elements per thread,
// 128 threads per 4096-element tile, 4 CTAs per SM.
//   thread (cp = tid % 8: columns 2cp, 2cp+1;  r = tid / 8)
//   exchange: float4 rows [..][8 pairs]; the transposing one (T1 A) in
//   8-byte elements, [s][kt][j2] with kt pitch 17 and s pitch 273 (both sides
//   conflict-free).
namespace pair {
constexpr int NT = 128;
constexpr int XB2 = 16 * 273;  // float2 elements of the exchange buffer (>= 4096)

__device__ __forceinline__ float4 ld16_hbm(const float2* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld16_l2(const float2* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st16(float2* p, float2 a, float2 b, uint64_t pol) {
  st_hint(reinterpret_cast<float4*>(p), make_float4(a.x, a.y, b.x, b.y), pol);
}
}  // namespace pair

template <int RB, bool T1>
__device__ __forceinline__ int pair_b_line(int task, int dl, int p, int q) {
  constexpr int QB = RB / 16, DB = 16 / QB;
  const int ja = p + 16 * q;
  if constexpr (T1)  // ring [j2l][ja][ks][kt]; task = (ks, jblk)
    return ((((task >> 4) * DB + dl) * RB + ja) * 16 + (task & 15)) * 16;
  else  // ring [kb][ja][lane]
    return ((task * DB + dl) * RB + ja) * 16;
}

// PF: the next tile is prefetched by TMA into a 32 KB landing buffer while
// this one is computed (3 CTAs per SM); otherwise tiles are loaded straight
// into registers (4 CTAs per SM).
template <int RB, bool T1, bool PF>
__global__ void __launch_bounds__(pair::NT, PF ? 3 : 4) lean_pair(const __grid_constant__ Args a) {
  using V = float2;
  constexpr int QB = RB / 16, DB = 16 / QB;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* const land = smraw;  // PF: 32 KB, 1024-aligned (128B-swizzled A boxes)
  unsigned char* const xbase = smraw + (PF ? 32768 : 0);
  V* xb = reinterpret_cast<V*>(xbase);
  float4* xq = reinterpret_cast<float4*>(xbase);
  V* w256 = xb + (T1 ? pair::XB2 : 4096);  // the plain exchange needs no padding
  V* wlo = w256 + 256;
  // T1 B tiles: the tile's four-step twiddle factors, built once per tile in fp64 (below)
  __shared__ double2 twc[T1 ? DB * 8 : 1], twq[T1 ? 16 : 1], tws[T1 ? DB : 1];
  __shared__ float2 twj[T1 ? DB : 1];
  __shared__ SchedShared shs;
  __shared__ __align__(8) uint64_t lbar;
  __shared__ int pf_sh[2];
  const int tid = threadIdx.x, cp = tid % 8, r = tid / 8;
#define SRC reinterpret_cast<const V*>(a.src)
#define DST reinterpret_cast<V*>(a.dst)
#define STG reinterpret_cast<V*>(a.stg)
  for (int i = tid; i < 256; i += pair::NT) {
    w256[i] = to_v(wroot(i, 256), 0.f);
    wlo[i] = to_v(wroot(i, a.R), 0.f);
  }
  if (PF && tid == 0) {
    mbar_init(&lbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pf_sh[0] = pf_sh[1] = 0;
  }
  Sched sc{&shs};
  sc.init(a);
  bool nf = false;
  uint32_t lphase = 0;
  int isB, g, task;
  // PF: one TMA for a whole tile (thread 0).  A: box {16 columns, 1, 256 rows}
  // of the pass input, 128-byte swizzled; B: the tile's lines of the ring
  // (T0: one contiguous 32 KB block; T1: box {16 kt, 1 ks, RB ja, DB columns}).
  auto issue = [&](int tb, int tg, int tt) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(&lbar, 32768);
    const uint64_t pol = policy_evict_first();
    if (!tb) {
      tma_load_3d(land, &a.mapA, tg * 16, tt, 0, &lbar, pol);
    } else if constexpr (T1) {
      tma_load_5d(land, &a.mapB, 0, tt & 15, 0, (tt >> 4) * DB, tg % a.nslots, &lbar, pol);
    } else {
      const V* src = STG + (int64_t)(tg % a.nslots) * a.slot_elems + (int64_t)(tt * DB) * RB * 16;
      bulk_g2s(land, src, 32768, &lbar, pol);
    }
  };
  while (sc.next(a, isB, g, task)) {
    V* sp = STG + (int64_t)(g % a.nslots) * a.slot_elems;
    V x[16], y[16];  // columns 2cp (x) and 2cp + 1 (y)
    if constexpr (PF) {
      if (tid == 0 && !pf_sh[sc.cb]) issue(isB, g, task);  // not prefetched (first tile, or late producers)
      mbar_wait(&lbar, lphase);
      lphase ^= 1;
      const float4* L = reinterpret_cast<const float4*>(land);
      if (isB) {  // [dl][ja][16 lanes] rows of 128 bytes
#pragma unroll
        for (int dl = 0; dl < DB; ++dl)
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            const float4 t = L[(dl * RB + r + 16 * q) * 8 + cp];
            x[dl * QB + q] = make_float2(t.x, t.y);
            y[dl * QB + q] = make_float2(t.z, t.w);
          }
      } else {  // [jb][16 columns], 16-byte chunk c of row jb at c ^ (jb & 7)
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int jb = r + 16 * t;
          const float4 u = L[jb * 8 + (cp ^ (jb & 7))];
          x[t] = make_float2(u.x, u.y);
          y[t] = make_float2(u.z, u.w);
        }
      }
      __syncthreads();  // the landing buffer is free
    } else if (isB) {
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const float4 t = pair::ld16_l2(sp + pair_b_line<RB, T1>(task, dl, r, q) + 2 * cp);
          x[dl * QB + q] = make_float2(t.x, t.y);
          y[dl * QB + q] = make_float2(t.z, t.w);
        }
    } else {  // A: jb = s + 16 t with s = r
      const uint64_t pol = policy_evict_first();
      const V* p0 = SRC + (int64_t)g * 16 + 2 * cp + a.LS * (int64_t)(task + RB * r);
      const int64_t step = a.LS * (int64_t)(RB * 16);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float4 u = pair::ld16_hbm(p0 + t * step, pol);
        x[t] = make_float2(u.x, u.y);
        y[t] = make_float2(u.z, u.w);
      }
    }
    sc.after_loads(a, isB, g);
    if constexpr (PF) {
      // thread 0, after the fence that acquired the probe of the next task's
      // producers: prefetch it when they are done (always for A tiles)
      if (tid == 0) {
        const int nb = sc.cb ^ 1;
        const bool ok = shs.pos[nb] < a.total && (!shs.isB[nb] || sc.nxt_val >= a.ntA);
        pf_sh[nb] = ok;
        if (ok) issue(shs.isB[nb], shs.g[nb], shs.task[nb]);
        pf_sh[sc.cb] = 0;  // this slot is re-published with the task after next
      }
    }
    if (isB) {
      // ---- B stage 0: W_R^(ja kb) (T0: one kb per dl, shared by the pair;
      // T1: kb = kt + 16 ks differs between the columns), QB-point DFTs
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        const int kb = T1 ? 2 * cp + 16 * (task & 15) : task * DB + dl;
        const int e0 = r * kb, es = 16 * kb;  // < R
        V w = cmul(w256[(e0 >> 8) * (256 / RB)], wlo[e0 & 255]);
        const V st = cmul(w256[(es >> 8) * (256 / RB)], wlo[es & 255]);
        if constexpr (T1) {
          const int e1 = e0 + r, es1 = es + 16;  // kb + 1
          V w1 = cmul(w256[(e1 >> 8) * (256 / RB)], wlo[e1 & 255]);
          const V st1 = cmul(w256[(es1 >> 8) * (256 / RB)], wlo[es1 & 255]);
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            x[dl * QB + q] = cmul(x[dl * QB + q], w);
            y[dl * QB + q] = cmul(y[dl * QB + q], w1);
            if (q + 1 < QB) {
              w = cmul(w, st);
              w1 = cmul(w1, st1);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            x[dl * QB + q] = cmul(x[dl * QB + q], w);
            y[dl * QB + q] = cmul(y[dl * QB + q], w);
            if (q + 1 < QB) w = cmul(w, st);
          }
        }
      }
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        reg_dft<float, QB>(x + dl * QB);
        reg_dft<float, QB>(y + dl * QB);
      }
      {  // W_RB^(p kq)
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < QB; ++k) {
          wp += r * (256 / RB);
          const V w = *wp;
#pragma unroll
          for (int dl = 0; dl < DB; ++dl) {
            x[dl * QB + P<QB>(k)] = cmul(x[dl * QB + P<QB>(k)], w);
            y[dl * QB + P<QB>(k)] = cmul(y[dl * QB + P<QB>(k)], w);
          }
        }
      }
      if constexpr (T1) {
        // W_N^(j2 k1), k1 = c + 256 QB kp, c = (2cp + 16 ks) + 256 kq, from exact integer
        // exponents in fp64 (north star c), factored so that a tile needs 10 DB + 16
        // sincospi instead of three per thread:
        //   twc[dl][cp] = W_N^(j2 (2cp + 16 ks)),  twq[dl][kq] = W_N^(j2 256 kq),
        //   tws[dl] = W_N^(j2 256 QB) (the recurrence step),  twj[dl] = W_N^(j2) (column kt + 1)
        const uint64_t N = (uint64_t)a.N;
        const int ks = task & 15;
        for (int i = tid; i < DB * 8 + 16 + 2 * DB; i += pair::NT) {
          int dl2, kind, idx;
          if (i < DB * 8) {
            kind = 0, dl2 = i >> 3, idx = i & 7;
          } else if (i < DB * 8 + 16) {
            kind = 1, dl2 = (i - DB * 8) / QB, idx = (i - DB * 8) % QB;
          } else {
            kind = 2 + ((i - DB * 8 - 16) >= DB), dl2 = (i - DB * 8 - 16) % DB, idx = 0;
          }
          const uint64_t jg = (uint64_t)(a.j2off + g * 16 + (task >> 4) * DB + dl2);  // global column
          const uint64_t m = kind == 0 ? (uint64_t)(2 * idx + 16 * ks) : kind == 1 ? (uint64_t)(256 * idx)
                             : kind == 2 ? (uint64_t)(256 * QB) : 1ull;
          const double2 w = wroot((int64_t)((jg * m) % N), a.N);
          if (kind == 0) twc[i] = w;
          else if (kind == 1) twq[i - DB * 8] = w;
          else if (kind == 2) tws[dl2] = w;
          else twj[dl2] = to_v(w, 0.f);
        }
      }
      // consumed staging lines: 8 threads share a line, thread cp drops the
      // lines of its loads cp and cp + 8
#pragma unroll
      for (int i = cp; i < 16; i += 8) l2_discard(sp + pair_b_line<RB, T1>(task, i / QB, r, i % QB));
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int k = 0; k < QB; ++k) {
          const V u = x[dl * QB + P<QB>(k)], w = y[dl * QB + P<QB>(k)];
          xq[((dl * QB + k) * 16 + r) * 8 + cp] = make_float4(u.x, u.y, w.x, w.y);
        }
    } else {
      // ---- A stage 0: 16-point DFTs over t, W_256^(s kt) shared by the pair
      if (a.check_finite) {
        // v * 0 is +-0 for a finite v and NaN for +-Inf / NaN: one FFMA2 per complex value
        // (four independent accumulators: the chain must not sit on the tile's critical path)
        const V zero = make_float2(0.f, 0.f);
        V acc[4] = {zero, zero, zero, zero};
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          acc[t & 1] = fma2(x[t], zero, acc[t & 1]);
          acc[2 + (t & 1)] = fma2(y[t], zero, acc[2 + (t & 1)]);
        }
        const V sum = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
        nf |= !(sum.x == 0.f && sum.y == 0.f);
      }
      if constexpr (T1) {
        if (a.cin.y != 1.0) {  // inverse: conjugate the input (forward: identity)
          const V ci = cvt(a.cin, 0.f);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            x[t] = mul2(x[t], ci);
            y[t] = mul2(y[t], ci);
          }
        }
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      {
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < 16; ++k) {
          wp += r;
          const V w = *wp;
          x[P<16>(k)] = cmul(x[P<16>(k)], w);
          y[P<16>(k)] = cmul(y[P<16>(k)], w);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if constexpr (T1) {  // [s][kt][j2]: s pitch 273, kt pitch 17
          xb[r * 273 + k * 17 + 2 * cp] = x[P<16>(k)];
          xb[r * 273 + k * 17 + 2 * cp + 1] = y[P<16>(k)];
        } else {  // [kt][s][pair]
          const V u = x[P<16>(k)], w = y[P<16>(k)];
          xq[(k * 16 + r) * 8 + cp] = make_float4(u.x, u.y, w.x, w.y);
        }
      }
    }
    sc.before_exchange(a, g);
    __syncthreads();
    if (isB) {
      // ---- B stage 1: 16-point DFTs over p; thread (cp, dl, kq)
      const int kq = r % QB, dl = r / QB;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float4 t = xq[((dl * QB + kq) * 16 + u) * 8 + cp];
        x[u] = make_float2(t.x, t.y);
        y[u] = make_float2(t.z, t.w);
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      const uint64_t pol = policy_evict_first();
      if constexpr (T1) {
        // y[k1 + R1 j2] = Y W_N^(j2 k1), k1 = kt + 16 ks + 256 kq + 256 QB kp, kt = 2cp (+1)
        const int j2 = g * 16 + (task >> 4) * DB + dl;
        const uint32_t c = (uint32_t)(2 * cp + 16 * (task & 15) + 256 * kq);
        // W_N^(j2 k1) for columns kt and kt + 1 from exact integer exponents:
        // fp64 bases and step (sincospi), fp64 recurrence, one rounding per
        // use -- fp64-accurate twiddles on the fp32 path, no table (north star c)
        // (column kt + 1: times W_N^j2 in fp32, <= 1.5 ulp)
        double2 w0 = cmul(twc[dl * 8 + cp], twq[dl * QB + kq]);
        const V wj = twj[dl];
        const double2 st = tws[dl];
        if (a.obl == 0) {  // y[k1 + R j2]: one base pointer, immediate offsets
          V* op = DST + (int64_t)j2 * a.R + c;
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) {
            const V w = to_v(w0, 0.f);
            pair::st16(op + kp * (256 * QB), cmul(x[P<16>(kp)], w), cmul(y[P<16>(kp)], cmul(w, wj)), pol);
            if (kp < 15) w0 = cmul(w0, st);
          }
        } else {  // sharded NCCL path: blocked by destination rank
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) {
            const V w = to_v(w0, 0.f);
            pair::st16(DST + t1_out(a, j2, c + kp * (256 * QB)), cmul(x[P<16>(kp)], w),
                       cmul(y[P<16>(kp)], cmul(w, wj)), pol);
            if (kp < 15) w0 = cmul(w0, st);
          }
        }
      } else {
        const int kb = task * DB + dl;
        const V co = cvt(a.cout, 0.f);
        V* op = DST + (int64_t)g * 16 + 2 * cp + a.LS * (int64_t)(kb + 256 * kq);
        const int64_t step = a.LS * (int64_t)(256 * QB);
        if (a.cout.x == 1.0 && a.cout.y == 1.0) {  // forward: no conjugation, no scale
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) pair::st16(op + kp * step, x[P<16>(kp)], y[P<16>(kp)], pol);
        } else {
#pragma unroll
          for (int kp = 0; kp < 16; ++kp)
            pair::st16(op + kp * step, mul2(x[P<16>(kp)], co), mul2(y[P<16>(kp)], co), pol);
        }
      }
    } else {
      // ---- A stage 1: 16-point DFTs over s -> ks, store to the ring
      // T0 thread (pair cp, kt = r): ring [kb][ja][lane], kb = kt + 16 ks
      // T1 thread (kt pair cp, j2l = r): ring [j2l][ja][ks][kt]
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if constexpr (T1) {
          x[u] = xb[u * 273 + (2 * cp) * 17 + r];
          y[u] = xb[u * 273 + (2 * cp + 1) * 17 + r];
        } else {
          const float4 t = xq[(r * 16 + u) * 8 + cp];
          x[u] = make_float2(t.x, t.y);
          y[u] = make_float2(t.z, t.w);
        }
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      const int base = T1 ? (r * RB + task) * 256 + 2 * cp : (r * RB + task) * 16 + 2 * cp;
      const int step = T1 ? 16 : 16 * RB * 16;
      const uint64_t keep = policy_evict_last();
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) pair::st16(sp + base + ks * step, x[P<16>(ks)], y[P<16>(ks)], keep);
    }
    sc.end(a, isB, g);
  }
  sc.finish(a, nf);
#undef SRC
#undef DST
#undef STG
}

// Pipelined complex64 tile kernel (EFFT_LEAN_PIPE): the paired kernel's tile
// arithmetic (32 points per thread, 128 threads per 32 KB tile) fed by TMA.
// One CTA per SM, 16 warps (all the register file holds at 128 registers):
//   * warps 0-11: three independent compute groups of 128 threads; group q owns
//     two 32 KB buffers: tile k + 1 lands in one while tile k is computed in the
//     other.  A group waits on the buffer's `full` mbarrier, reads its stage-0
//     points from it (A tiles: 128-byte-swizzled rows), uses the SAME buffer
//     for the exchange between the two radix stages (the transposing exchange
//     of the T1 A tile is XOR-swizzled, [s][kt][j2 pair ^ (kt >> 1)], so it
//     fits 32 KB without padding, both sides conflict-free), arrives on `empty`
//     once its stage-1 operands are in registers, stores from registers and
//     arrives on `done`.  Two 128-thread named barriers per tile; no CTA-wide
//     barrier, no fence, no atomic and no dependency probe in a compute warp.
//   * warps 12-14, lane 0: issue lanes, one per group (a blocked dependency
//     probe of one never delays another).  Static schedule: group
//     q of CTA c runs positions v, v + 3G, v + 6G, ... of the claim order
//     (v = c + q G, G = grid; all CTAs resident), so only the tiles in the
//     buffers are in flight and the staging ring stays L2-resident (a claim
//     counter running ahead widens the window of open groups).  A lane probes
//     the next position's dependency counter (ld.acquire) one tile ahead and
//     issues the tile with ONE TMA instruction the moment its buffer is free.
//   * warp 15, lane 0: the release lane: `done` seen (any group) -> ONE
//     fence.acq_rel (the tiles' stores, observed through the mbarriers, become
//     visible GPU-wide) -> a red per tile on its group's completion counter.
//     Its fence never delays an issue.  Nothing in either loop blocks, positions increase per group and
//     every dependency points backwards: the header's deadlock-freedom argument
//     holds unchanged.
namespace pipe {
constexpr int NG = 3;                 // compute groups
constexpr int NC = 128;               // threads per group
constexpr int NT = NG * NC + 128;     // + three issue warps (one lane each) and the release warp
constexpr int BUF = 32768;
struct Desc {
  int isB, g, task, pad;
  long long t_issue;  // dev profiling (EFFT_PIPE_ABL bit 256)
};
struct Group {
  uint64_t full[2], empty[2], done[4];  // done: a ring of 4 so an unobserved phase is never overrun
  Desc desc[2];
  int32_t* pend[4];                 // issue lane -> release lane: the completion counter of tile k (k & 3)
  volatile int ntiles;              // issue lane -> release lane: tiles issued in all (-1 while running)
  volatile uint32_t released;       // release lane -> issue lane: tiles published
  long long t_empty[2], t_done[4];  // dev profiling
};
struct Shared {
  Group grp[NG];
};
constexpr int SMEM = 2 * NG * BUF + 512 * 8 + (int)sizeof(Shared);
__device__ __forceinline__ void bar_compute(int q) { asm volatile("bar.sync %0, 128;" ::"r"(q + 1) : "memory"); }
}  // namespace pipe

// dev ablations (EFFT_PIPE_ABL bits, timing only -- results are wrong): 1 no arithmetic,
// 2 no global stores (32 / 64: no ring / no output stores), 4 no exchange, 8 no TMA loads,
// 16 no four-step twiddle, 256 cycle counters, 512 no dependencies, 1024 no release fence
#define ABL(bit) ((a.abl & (bit)) != 0)
template <int RB, bool T1>
__global__ void __launch_bounds__(pipe::NT, 1) lean_pipe(const __grid_constant__ Args a) {
  using V = float2;
  constexpr int QB = RB / 16, DB = 16 / QB;
  extern __shared__ __align__(1024) unsigned char smraw[];
  V* w256 = reinterpret_cast<V*>(smraw + 2 * pipe::NG * pipe::BUF);
  V* wlo = w256 + 256;
  pipe::Shared* shs = reinterpret_cast<pipe::Shared*>(wlo + 256);
#define SRC reinterpret_cast<const V*>(a.src)
#define DST reinterpret_cast<V*>(a.dst)
#define STG reinterpret_cast<V*>(a.stg)
  for (int i = threadIdx.x; i < 256; i += pipe::NT) {
    w256[i] = to_v(wroot(i, 256), 0.f);
    wlo[i] = to_v(wroot(i, a.R), 0.f);
  }
  if (threadIdx.x < pipe::NG) {
    pipe::Group* sh = &shs->grp[threadIdx.x];
    sh->ntiles = -1;
    sh->released = 0;
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sh->full[i], 1);
      mbar_init(&sh->empty[i], pipe::NC);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&sh->done[i], pipe::NC);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= pipe::NG * pipe::NC + 96) {
    // ---------------- release lane ----------------
    // One lane for the three groups: every `done` seen in a sweep is published
    // behind ONE fence.acq_rel (the tiles' stores, observed through the
    // mbarriers, become visible GPU-wide), then one red per tile on its group's
    // completion counter.  `released` tells the issue lanes how far it got, so
    // the `done` / pend rings are never overrun.
    if (threadIdx.x != pipe::NG * pipe::NC + 96) return;
    uint32_t kr[pipe::NG] = {0, 0, 0}, kn[pipe::NG];
    long long idle = 0;
    for (;;) {
      bool any = false, fin = true;
#pragma unroll
      for (int q = 0; q < pipe::NG; ++q) {
        pipe::Group* sh = &shs->grp[q];
        kn[q] = kr[q];
        while (kn[q] - kr[q] < 3 && mbar_test(&sh->done[kn[q] & 3], (kn[q] >> 2) & 1)) ++kn[q];
        any |= kn[q] != kr[q];
        const int nt = sh->ntiles;
        fin &= nt >= 0 && kn[q] == (uint32_t)nt;
      }
      if (any) {
        if (!ABL(1024)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
        for (int q = 0; q < pipe::NG; ++q) {
          pipe::Group* sh = &shs->grp[q];
          for (; kr[q] != kn[q]; ++kr[q])
            asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(sh->pend[kr[q] & 3]) : "memory");
          sh->released = kr[q];
        }
        idle = 0;
      } else if (fin) {
        break;
      } else {
        __nanosleep(64);
        if (++idle == (1ll << 24)) {
          printf("EFFT lean pipe release lane stuck cta=%d kr=%u %u %u\n", blockIdx.x, kr[0], kr[1], kr[2]);
          __trap();
        }
      }
    }
    return;
  }
  if (threadIdx.x >= pipe::NG * pipe::NC) {
    // ---------------- issue lanes (lane 0 of warps 12, 13, 14) ----------------
    if (threadIdx.x % 32 != 0) return;
    const int q = (threadIdx.x - pipe::NG * pipe::NC) / 32;
    pipe::Group* sh = &shs->grp[q];
    unsigned char* const bufs = smraw + q * 2 * pipe::BUF;
    const uint64_t pol = policy_evict_first();
    struct Task {
      long long pos;
      int isB, g, task, val, need;
    };
    auto probe = [&](const Task& t) -> int {
      if (t.isB) return ld_acquire(a.doneA + t.g);        // B(g) needs A(g) complete
      if (t.g < a.nslots) return a.ntB;
      return ld_acquire(a.doneB + (t.g - a.nslots));      // A(g) stores into the slot B(g - nslots) read
    };
    auto setup = [&](Task& t, long long pos) {
      t.pos = pos;
      t.isB = t.g = t.task = 0;
      t.val = t.need = 0;
      if (pos < a.total) {
        decode(a, (uint32_t)pos, t.isB, t.g, t.task);
        t.need = t.isB ? a.ntA : a.ntB;
        t.val = probe(t);
      }
    };
    const long long G = (long long)gridDim.x * pipe::NG, v = blockIdx.x + (long long)q * gridDim.x;
    Task cur, nxt;
    setup(cur, v);
    setup(nxt, v + G);
    uint32_t ki = 0, ke = 0;  // tiles issued / buffer freed
    long long idle = 0, late = 0, obs_e = 0, iss_d = 0, t_obs[2] = {0, 0};
    for (;;) {
      bool prog = false;
      while (ke < ki && mbar_test(&sh->empty[ke & 1], (ke >> 1) & 1)) {
        if (ABL(256)) {
          t_obs[ke & 1] = clock64();
          obs_e += t_obs[ke & 1] - sh->t_empty[ke & 1];
        }
        ++ke;
        prog = true;
      }
      // (ki - released < 4: the `done` ring and the pend ring are never overrun)
      if (ki - ke < 2 && ki - sh->released < 4) {
        const int b = ki & 1;
        if (cur.pos >= a.total) {
          sh->desc[b].isB = -1;
          mbar_arrive(&sh->full[b]);
          sh->ntiles = (int)ki;
          if (ABL(256) && blockIdx.x < 2)
            printf("pipe prof cta %d group %d issue lane: tiles %u, late deps %lld, empty arrive->seen %lld, "
                   "seen->issue %lld\n", blockIdx.x, q, ki, late, obs_e / (ki ? ki : 1), iss_d / (ki ? ki : 1));
          break;
        }
        if (ABL(512)) cur.val = cur.need;
        if (cur.val < cur.need) {  // the producers of this tile are late
          cur.val = probe(cur);
          ++late;
        }
        if (cur.val >= cur.need) {
          sh->desc[b].isB = cur.isB;
          sh->desc[b].g = cur.g;
          sh->desc[b].task = cur.task;
          sh->pend[ki & 3] = cur.isB ? a.doneB + cur.g : a.doneA + cur.g;
          if (ABL(256)) {
            sh->desc[b].t_issue = clock64();
            if (ki >= 2) iss_d += sh->desc[b].t_issue - t_obs[b];
          }
          unsigned char* land = bufs + b * pipe::BUF;
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (ABL(8)) {
            mbar_arrive(&sh->full[b]);
          } else {
            mbar_arrive_tx(&sh->full[b], pipe::BUF);
            if (!cur.isB) {
              tma_load_3d(land, &a.mapA, cur.g * 16, cur.task, 0, &sh->full[b], pol);
            } else if constexpr (T1) {
              tma_load_5d(land, &a.mapB, 0, cur.task & 15, 0, (cur.task >> 4) * DB, cur.g % a.nslots, &sh->full[b],
                          pol);
            } else {
              const V* src = STG + (int64_t)(cur.g % a.nslots) * a.slot_elems + (int64_t)(cur.task * DB) * RB * 16;
              bulk_g2s(land, src, pipe::BUF, &sh->full[b], pol);
            }
          }
          ++ki;
          cur = nxt;
          setup(nxt, v + (long long)(ki + 1) * G);
          prog = true;
        }
      }
      if (!prog) {
        __nanosleep(a.abl >> 16 ? (a.abl >> 16) : 64);
        if (++idle == (1ll << 24)) {
          printf("EFFT lean pipe issue lane stuck cta=%d q=%d pos=%lld isB=%d g=%d task=%d ki=%u ke=%u released=%u\n",
                 blockIdx.x, q, cur.pos, cur.isB, cur.g, cur.task, ki, ke, sh->released);
          __trap();
        }
      } else {
        idle = 0;
      }
    }
    return;
  }
  // ---------------- compute warps ----------------
  const int q = threadIdx.x / pipe::NC, tid = threadIdx.x % pipe::NC;
  // T1 B tiles: the tile's four-step twiddle factors, built once per tile in fp64 (as in lean_pair)
  __shared__ double2 twc_[pipe::NG][T1 ? DB * 8 : 1], twq_[pipe::NG][T1 ? 16 : 1], tws_[pipe::NG][T1 ? DB : 1];
  __shared__ float2 twj_[pipe::NG][T1 ? DB : 1];
  double2* const twc = twc_[q];
  double2* const twq = twq_[q];
  double2* const tws = tws_[q];
  float2* const twj = twj_[q];
  pipe::Group* sh = &shs->grp[q];
  unsigned char* const bufs = smraw + q * 2 * pipe::BUF;
  const int cp = tid % 8, r = tid / 8;
  bool nf = false;
  long long pw = 0, pl = 0, pt0 = clock64(), pn = 0;  // dev profiling
  for (uint32_t k = 0;; ++k) {
    const int b = k & 1;
    const long long tw = ABL(256) ? clock64() : 0;
    mbar_wait(&sh->full[b], (k >> 1) & 1);
    const int isB = sh->desc[b].isB;
    if (isB < 0) break;
    if (ABL(256)) {
      const long long tn = clock64();
      pw += tn - tw;
      pl += tn - sh->desc[b].t_issue;
      ++pn;
    }
    const int g = sh->desc[b].g, task = sh->desc[b].task;
    V* sp = STG + (int64_t)(g % a.nslots) * a.slot_elems;
    unsigned char* const buf = bufs + b * pipe::BUF;
    V* xb = reinterpret_cast<V*>(buf);
    float4* xq = reinterpret_cast<float4*>(buf);
    V x[16], y[16];  // columns 2cp (x) and 2cp + 1 (y)
    if (isB) {  // [dl][ja][16 lanes] rows of 128 bytes
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const float4 t = xq[(dl * RB + r + 16 * q) * 8 + cp];
          x[dl * QB + q] = make_float2(t.x, t.y);
          y[dl * QB + q] = make_float2(t.z, t.w);
        }
    } else {  // [jb][16 columns], 16-byte chunk c of row jb at c ^ (jb & 7); jb = r + 16 t
      const float4* L = xq + r * 8 + (cp ^ (r & 7));
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float4 u = L[t * 128];
        x[t] = make_float2(u.x, u.y);
        y[t] = make_float2(u.z, u.w);
      }
    }
    if (!ABL(4)) pipe::bar_compute(q);  // every thread has its points: the buffer becomes the exchange
    if (ABL(1)) {
    } else if (isB) {
      // ---- B stage 0: W_R^(ja kb), QB-point DFTs
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        const int kb = T1 ? 2 * cp + 16 * (task & 15) : task * DB + dl;
        const int e0 = r * kb, es = 16 * kb;  // < R
        V w = cmul(w256[(e0 >> 8) * (256 / RB)], wlo[e0 & 255]);
        const V st = cmul(w256[(es >> 8) * (256 / RB)], wlo[es & 255]);
        if constexpr (T1) {
          const int e1 = e0 + r, es1 = es + 16;  // kb + 1
          V w1 = cmul(w256[(e1 >> 8) * (256 / RB)], wlo[e1 & 255]);
          const V st1 = cmul(w256[(es1 >> 8) * (256 / RB)], wlo[es1 & 255]);
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            x[dl * QB + q] = cmul(x[dl * QB + q], w);
            y[dl * QB + q] = cmul(y[dl * QB + q], w1);
            if (q + 1 < QB) {
              w = cmul(w, st);
              w1 = cmul(w1, st1);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            x[dl * QB + q] = cmul(x[dl * QB + q], w);
            y[dl * QB + q] = cmul(y[dl * QB + q], w);
            if (q + 1 < QB) w = cmul(w, st);
          }
        }
      }
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        reg_dft<float, QB>(x + dl * QB);
        reg_dft<float, QB>(y + dl * QB);
      }
      {  // W_RB^(p kq)
        const V* wp = w256;
#pragma unroll
        for (int k2 = 1; k2 < QB; ++k2) {
          wp += r * (256 / RB);
          const V w = *wp;
#pragma unroll
          for (int dl = 0; dl < DB; ++dl) {
            x[dl * QB + P<QB>(k2)] = cmul(x[dl * QB + P<QB>(k2)], w);
            y[dl * QB + P<QB>(k2)] = cmul(y[dl * QB + P<QB>(k2)], w);
          }
        }
      }
    } else {
      // ---- A stage 0: 16-point DFTs over t, W_256^(s kt) shared by the pair
      if (a.check_finite) {
        // v * 0 is +-0 for a finite v and NaN for +-Inf / NaN: one FFMA2 per complex value
        // (four independent accumulators: the chain must not sit on the tile's critical path)
        const V zero = make_float2(0.f, 0.f);
        V acc[4] = {zero, zero, zero, zero};
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          acc[t & 1] = fma2(x[t], zero, acc[t & 1]);
          acc[2 + (t & 1)] = fma2(y[t], zero, acc[2 + (t & 1)]);
        }
        const V sum = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
        nf |= !(sum.x == 0.f && sum.y == 0.f);
      }
      if constexpr (T1) {
        if (a.cin.y != 1.0) {  // inverse: conjugate the input (forward: identity)
          const V ci = cvt(a.cin, 0.f);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            x[t] = mul2(x[t], ci);
            y[t] = mul2(y[t], ci);
          }
        }
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      {
        const V* wp = w256;
#pragma unroll
        for (int k2 = 1; k2 < 16; ++k2) {
          wp += r;
          const V w = *wp;
          x[P<16>(k2)] = cmul(x[P<16>(k2)], w);
          y[P<16>(k2)] = cmul(y[P<16>(k2)], w);
        }
      }
    }
    if (ABL(4)) {
    } else if (isB) {
      if constexpr (T1) {  // twc[dl][cp], twq[dl][kq], tws[dl], twj[dl]: see lean_pair
        const uint64_t N = (uint64_t)a.N;
        const int ks = task & 15;
        for (int i = tid; i < DB * 8 + 16 + 2 * DB; i += pipe::NC) {
          int dl2, kind, idx;
          if (i < DB * 8) {
            kind = 0, dl2 = i >> 3, idx = i & 7;
          } else if (i < DB * 8 + 16) {
            kind = 1, dl2 = (i - DB * 8) / QB, idx = (i - DB * 8) % QB;
          } else {
            kind = 2 + ((i - DB * 8 - 16) >= DB), dl2 = (i - DB * 8 - 16) % DB, idx = 0;
          }
          const uint64_t jg = (uint64_t)(a.j2off + g * 16 + (task >> 4) * DB + dl2);  // global column
          const uint64_t m = kind == 0 ? (uint64_t)(2 * idx + 16 * ks) : kind == 1 ? (uint64_t)(256 * idx)
                             : kind == 2 ? (uint64_t)(256 * QB) : 1ull;
          const double2 w = wroot((int64_t)((jg * m) % N), a.N);
          if (kind == 0) twc[i] = w;
          else if (kind == 1) twq[i - DB * 8] = w;
          else if (kind == 2) tws[dl2] = w;
          else twj[dl2] = to_v(w, 0.f);
        }
      }
      // the consumed staging lines leave L2 without write-back
#pragma unroll
      for (int i = cp; i < 16; i += 8) l2_discard(sp + pair_b_line<RB, T1>(task, i / QB, r, i % QB));
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int k2 = 0; k2 < QB; ++k2) {
          const V u = x[dl * QB + P<QB>(k2)], w = y[dl * QB + P<QB>(k2)];
          xq[((dl * QB + k2) * 16 + r) * 8 + cp] = make_float4(u.x, u.y, w.x, w.y);
        }
    } else {
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const V u = x[P<16>(k2)], w = y[P<16>(k2)];
        if constexpr (T1)  // [s][kt][j2 pair ^ (kt >> 1)]
          xq[r * 128 + k2 * 8 + (cp ^ (k2 >> 1))] = make_float4(u.x, u.y, w.x, w.y);
        else  // [kt][s][pair]
          xq[(k2 * 16 + r) * 8 + cp] = make_float4(u.x, u.y, w.x, w.y);
      }
    }
    if (!ABL(4)) pipe::bar_compute(q);
    if (isB) {
      // ---- B stage 1: 16-point DFTs over p; thread (cp, dl, kq)
      const int kq = r % QB, dl = r / QB;
      if (!ABL(4)) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float4 t = xq[((dl * QB + kq) * 16 + u) * 8 + cp];
        x[u] = make_float2(t.x, t.y);
        y[u] = make_float2(t.z, t.w);
      }
      }
      if (ABL(256) && tid == 0) sh->t_empty[b] = clock64();
      mbar_arrive(&sh->empty[b]);  // stage-1 operands are in registers: the buffer is free
      if (!ABL(1)) {
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      }
      const uint64_t pol = policy_evict_first();
      if constexpr (T1) {
        // y[k1 + R1 j2] = Y W_N^(j2 k1), k1 = kt + 16 ks + 256 kq + 256 QB kp, kt = 2cp (+1)
        const int j2 = g * 16 + (task >> 4) * DB + dl;
        const uint32_t c = (uint32_t)(2 * cp + 16 * (task & 15) + 256 * kq);
        // exact integer exponents, fp64 bases and step, fp64 recurrence (see lean_pair)
        double2 w0 = cmul(twc[dl * 8 + cp], twq[dl * QB + kq]);
        const V wj = twj[dl];
        const double2 st = tws[dl];
        if (ABL(2) || ABL(64)) {
        } else if (ABL(128)) {  // timing experiment: the same bytes as 256-byte segments
          const int ks = task & 15;
          V* op = DST + (int64_t)(g * 16 + (task >> 4) * DB + (ks & 1)) * a.R + 2 * cp + 16 * (r & 1) + 32 * (ks >> 1) +
                  256 * ((r >> 1) & (QB - 1));
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) pair::st16(op + kp * (256 * QB), x[P<16>(kp)], y[P<16>(kp)], pol);
        } else if (ABL(16)) {
          V* op = DST + (int64_t)j2 * a.R + c;
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) pair::st16(op + kp * (256 * QB), x[P<16>(kp)], y[P<16>(kp)], pol);
        } else if (a.obl == 0) {
          V* op = DST + (int64_t)j2 * a.R + c;
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) {
            const V w = to_v(w0, 0.f);
            pair::st16(op + kp * (256 * QB), cmul(x[P<16>(kp)], w), cmul(y[P<16>(kp)], cmul(w, wj)), pol);
            if (kp < 15) w0 = cmul(w0, st);
          }
        } else {
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) {
            const V w = to_v(w0, 0.f);
            pair::st16(DST + t1_out(a, j2, c + kp * (256 * QB)), cmul(x[P<16>(kp)], w),
                       cmul(y[P<16>(kp)], cmul(w, wj)), pol);
            if (kp < 15) w0 = cmul(w0, st);
          }
        }
      } else {
        const int kb = task * DB + dl;
        const V co = cvt(a.cout, 0.f);
        V* op = DST + (int64_t)g * 16 + 2 * cp + a.LS * (int64_t)(kb + 256 * kq);
        if (ABL(128))  // timing experiment: the same bytes as 256-byte segments
          op = DST + (int64_t)(g >> 1) * 32 + 16 * (r & 1) + 2 * cp +
               a.LS * (int64_t)(task * DB + (g & 1) + 256 * ((r >> 1) & (QB - 1)));
        const int64_t step = a.LS * (int64_t)(256 * QB);
        if (ABL(2) || ABL(64)) {
        } else if (a.cout.x == 1.0 && a.cout.y == 1.0) {  // forward: no conjugation, no scale
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) pair::st16(op + kp * step, x[P<16>(kp)], y[P<16>(kp)], pol);
        } else {
#pragma unroll
          for (int kp = 0; kp < 16; ++kp)
            pair::st16(op + kp * step, mul2(x[P<16>(kp)], co), mul2(y[P<16>(kp)], co), pol);
        }
      }
    } else {
      // ---- A stage 1: 16-point DFTs over s -> ks, store to the ring
      // T0 thread (pair cp, kt = r): ring [kb][ja][lane], kb = kt + 16 ks
      // T1 thread (kt pair cp, j2l = r): ring [j2l][ja][ks][kt]
      if (ABL(4)) {
      } else if constexpr (T1) {
        const V* L = xb + (2 * cp) * 16 + (((r >> 1) ^ cp) & 7) * 2 + (r & 1);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          x[u] = L[u * 256];
          y[u] = L[u * 256 + 16];
        }
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float4 t = xq[(r * 16 + u) * 8 + cp];
          x[u] = make_float2(t.x, t.y);
          y[u] = make_float2(t.z, t.w);
        }
      }
      if (ABL(256) && tid == 0) sh->t_empty[b] = clock64();
      mbar_arrive(&sh->empty[b]);
      if (!ABL(1)) {
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      }
      const int base = T1 ? (r * RB + task) * 256 + 2 * cp : (r * RB + task) * 16 + 2 * cp;
      const int step = T1 ? 16 : 16 * RB * 16;
      const uint64_t keep = policy_evict_last();
      if (!ABL(2) && !ABL(32)) {
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) pair::st16(sp + base + ks * step, x[P<16>(ks)], y[P<16>(ks)], keep);
      }
    }
    if (ABL(256) && tid == 0) sh->t_done[k & 3] = clock64();
    mbar_arrive(&sh->done[k & 3]);  // stores issued
  }
  if (ABL(256) && tid == 0 && blockIdx.x < 2 && pn)
    printf("pipe prof cta %d compute: %lld tiles, %lld cycles per tile, waiting for the tile %lld, issue->ready %lld\n",
           blockIdx.x, pn, (clock64() - pt0) / pn, pw / pn, pl / pn);
  if (__any_sync(0xffffffffu, nf) && (tid & 31) == 0) atomicOr(a.flag, 1);
#undef SRC
#undef DST
#undef STG
}

// Wide complex64 tile kernel: F = 32 columns per group, so every HBM access
// is a 256-byte segment (tools/skel_bench.cu: a strided read + strided write
// pass reaches 5.9 TB/s with 256-byte segments vs 4.4 TB/s with 128-byte
// ones).  64 KB tiles, 256 threads, 32 points per thread (two adjacent
// columns, 16-byte lanes), one 64 KB shared-memory exchange per sub-stage,
// two CTAs per SM; scheduling as lean_pair (Sched).
//   A tile:  thread (column pair cp < 16, s < 16), rows jb = s + 16 t
//   T0 B:    ring [kb][ja][32 lanes], tile = DB kb x RB ja x 32 columns
//   T1 B:    ring [j2l][ja][ks][kt], tile = 2 ks x 16 kt x RB ja x DB columns,
//            task = (ks pair ksp, column block jblk): 32 consecutive k1 per column
namespace wide {
constexpr int NT = 256;
constexpr int KP = 33, SP = 16 * KP + 1;  // float2 pitches of the transposing A exchange [s][kt][j2]
constexpr int XB1 = 16 * SP;              // 8464 float2
constexpr int SMEM_T1 = XB1 * 8 + 512 * 8;
constexpr int SMEM_T0 = 8192 * 8 + 512 * 8;
}  // namespace wide

template <int RB, bool T1>
__device__ __forceinline__ int wide_b_line(int task, int dl, int p, int q, int ksl) {
  constexpr int QB = RB / 16, DB = 16 / QB;
  const int ja = p + 16 * q;
  if constexpr (T1)  // ring [j2l][ja][ks][kt]; task = (ksp = task & 7, jblk = task >> 3)
    return ((((task >> 3) * DB + dl) * RB + ja) * 16 + 2 * (task & 7) + ksl) * 16;
  else  // ring [kb][ja][32 lanes]
    return ((task * DB + dl) * RB + ja) * 32;
}

template <int RB, bool T1>
__global__ void __launch_bounds__(wide::NT, 2) lean_wide(const __grid_constant__ Args a) {
  using V = float2;
  constexpr int QB = RB / 16, DB = 16 / QB;
  extern __shared__ __align__(128) unsigned char smraw[];
  V* xb = reinterpret_cast<V*>(smraw);
  float4* xq = reinterpret_cast<float4*>(smraw);
  V* w256 = xb + (T1 ? wide::XB1 : 8192);
  V* wlo = w256 + 256;
  __shared__ SchedShared shs;
  const int tid = threadIdx.x;
#define SRC reinterpret_cast<const V*>(a.src)
#define DST reinterpret_cast<V*>(a.dst)
#define STG reinterpret_cast<V*>(a.stg)
  for (int i = tid; i < 256; i += wide::NT) {
    w256[i] = to_v(wroot(i, 256), 0.f);
    wlo[i] = to_v(wroot(i, a.R), 0.f);
  }
  Sched sc{&shs};
  sc.init(a);
  bool nf = false;
  int isB, g, task;
  while (sc.next(a, isB, g, task)) {
    V* sp = STG + (int64_t)(g % a.nslots) * a.slot_elems;
    V x[16], y[16];  // columns 2cp (x) and 2cp + 1 (y)
    // thread roles
    //   A: T0 cp = tid & 15, s = tid >> 4;  T1 (bank-conflict-free STS.64 halves):
    //      cp = (tid & 7) + 8 ((tid >> 5) & 1), s = 4 (tid >> 6) + ((tid >> 3) & 3)
    //   B: T0 cp = tid & 15, p = tid >> 4;  T1 cp = tid & 7 (kt pair), ksl = (tid >> 3) & 1, p = tid >> 4
    int cp, r, ksl = 0;
    if (!isB) {
      if constexpr (T1) {
        cp = (tid & 7) + 8 * ((tid >> 5) & 1);
        r = 4 * (tid >> 6) + ((tid >> 3) & 3);
      } else {
        cp = tid & 15;
        r = tid >> 4;
      }
    } else {
      if constexpr (T1) {
        cp = tid & 7;
        ksl = (tid >> 3) & 1;
      } else {
        cp = tid & 15;
      }
      r = tid >> 4;
    }
    if (isB) {
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const float4 t = pair::ld16_l2(sp + wide_b_line<RB, T1>(task, dl, r, q, ksl) + 2 * cp);
          x[dl * QB + q] = make_float2(t.x, t.y);
          y[dl * QB + q] = make_float2(t.z, t.w);
        }
    } else {  // A: jb = s + 16 t with s = r
      const uint64_t pol = policy_evict_first();
      const V* p0 = SRC + (int64_t)g * 32 + 2 * cp + a.LS * (int64_t)(task + RB * r);
      const int64_t step = a.LS * (int64_t)(RB * 16);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float4 u = pair::ld16_hbm(p0 + t * step, pol);
        x[t] = make_float2(u.x, u.y);
        y[t] = make_float2(u.z, u.w);
      }
    }
    sc.after_loads(a, isB, g);
    if (isB) {
      // ---- B stage 0: W_R^(ja kb), QB-point DFTs over q
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        const int kb = T1 ? 2 * cp + 16 * (2 * (task & 7) + ksl) : task * DB + dl;
        const int e0 = r * kb, es = 16 * kb;  // < R
        V w = cmul(w256[(e0 >> 8) * (256 / RB)], wlo[e0 & 255]);
        const V st = cmul(w256[(es >> 8) * (256 / RB)], wlo[es & 255]);
        if constexpr (T1) {
          const int e1 = e0 + r, es1 = es + 16;  // kb + 1
          V w1 = cmul(w256[(e1 >> 8) * (256 / RB)], wlo[e1 & 255]);
          const V st1 = cmul(w256[(es1 >> 8) * (256 / RB)], wlo[es1 & 255]);
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            x[dl * QB + q] = cmul(x[dl * QB + q], w);
            y[dl * QB + q] = cmul(y[dl * QB + q], w1);
            if (q + 1 < QB) {
              w = cmul(w, st);
              w1 = cmul(w1, st1);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            x[dl * QB + q] = cmul(x[dl * QB + q], w);
            y[dl * QB + q] = cmul(y[dl * QB + q], w);
            if (q + 1 < QB) w = cmul(w, st);
          }
        }
      }
#pragma unroll
      for (int dl = 0; dl < DB; ++dl) {
        reg_dft<float, QB>(x + dl * QB);
        reg_dft<float, QB>(y + dl * QB);
      }
      {  // W_RB^(p kq)
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < QB; ++k) {
          wp += r * (256 / RB);
          const V w = *wp;
#pragma unroll
          for (int dl = 0; dl < DB; ++dl) {
            x[dl * QB + P<QB>(k)] = cmul(x[dl * QB + P<QB>(k)], w);
            y[dl * QB + P<QB>(k)] = cmul(y[dl * QB + P<QB>(k)], w);
          }
        }
      }
      // consumed staging lines leave L2 without write-back: a 128-byte line is
      // read by the 8 lanes of one warp; each of them drops two
      {
        const int own = cp & 7, half = T1 ? 0 : (cp >> 3);
#pragma unroll
        for (int i = own; i < 16; i += 8) l2_discard(sp + wide_b_line<RB, T1>(task, i / QB, r, i % QB, ksl) + 16 * half);
      }
#pragma unroll
      for (int dl = 0; dl < DB; ++dl)
#pragma unroll
        for (int k = 0; k < QB; ++k) {
          const V u = x[dl * QB + P<QB>(k)], w = y[dl * QB + P<QB>(k)];
          if constexpr (T1)  // [ksl][dl][kq][p][8 kt pairs]
            xq[(((ksl * DB + dl) * QB + k) * 16 + r) * 8 + cp] = make_float4(u.x, u.y, w.x, w.y);
          else  // [dl][kq][p][16 pairs]
            xq[((dl * QB + k) * 16 + r) * 16 + cp] = make_float4(u.x, u.y, w.x, w.y);
        }
    } else {
      // ---- A stage 0: 16-point DFTs over t, W_256^(s kt) shared by the pair
      if (a.check_finite) {
        // v * 0 is +-0 for a finite v and NaN for +-Inf / NaN: one FFMA2 per complex value
        // (four independent accumulators: the chain must not sit on the tile's critical path)
        const V zero = make_float2(0.f, 0.f);
        V acc[4] = {zero, zero, zero, zero};
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          acc[t & 1] = fma2(x[t], zero, acc[t & 1]);
          acc[2 + (t & 1)] = fma2(y[t], zero, acc[2 + (t & 1)]);
        }
        const V sum = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
        nf |= !(sum.x == 0.f && sum.y == 0.f);
      }
      if constexpr (T1) {
        if (a.cin.y != 1.0) {  // inverse: conjugate the input (forward: identity)
          const V ci = cvt(a.cin, 0.f);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            x[t] = mul2(x[t], ci);
            y[t] = mul2(y[t], ci);
          }
        }
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      {
        const V* wp = w256;
#pragma unroll
        for (int k = 1; k < 16; ++k) {
          wp += r;
          const V w = *wp;
          x[P<16>(k)] = cmul(x[P<16>(k)], w);
          y[P<16>(k)] = cmul(y[P<16>(k)], w);
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if constexpr (T1) {  // [s][kt][j2]: s pitch SP, kt pitch KP (odd: two STS.64)
          xb[r * wide::SP + k * wide::KP + 2 * cp] = x[P<16>(k)];
          xb[r * wide::SP + k * wide::KP + 2 * cp + 1] = y[P<16>(k)];
        } else {  // [kt][s][16 pairs]
          const V u = x[P<16>(k)], w = y[P<16>(k)];
          xq[(k * 16 + r) * 16 + cp] = make_float4(u.x, u.y, w.x, w.y);
        }
      }
    }
    sc.before_exchange(a, g);
    __syncthreads();
    if (isB) {
      // ---- B stage 1: 16-point DFTs over p; thread (cp, [ksl], dl, kq), r = tid >> 4
      const int kq = r % QB, dl = r / QB;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float4 t = T1 ? xq[(((ksl * DB + dl) * QB + kq) * 16 + u) * 8 + cp] : xq[((dl * QB + kq) * 16 + u) * 16 + cp];
        x[u] = make_float2(t.x, t.y);
        y[u] = make_float2(t.z, t.w);
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      const uint64_t pol = policy_evict_first();
      if constexpr (T1) {
        // y[k1 + R1 j2] = Y W_N^(j2 k1), k1 = kt + 16 ks + 256 kq + 256 QB kp, kt = 2cp (+1), ks = 2 ksp + ksl
        const int j2 = g * 32 + (task >> 3) * DB + dl;
        const uint32_t c = (uint32_t)(2 * cp + 16 * (2 * (task & 7) + ksl) + 256 * kq);
        // W_N^(j2 k1): fp64 base and step from exact exponents, fp64 recurrence, one rounding per use
        const uint64_t N = (uint64_t)a.N, jg = (uint64_t)(a.j2off + j2);
        double2 w0 = wroot((int64_t)((jg * c) % N), a.N);
        const V wj = to_v(wroot((int64_t)(jg % N), a.N), 0.f);
        const double2 st = wroot((int64_t)((jg * (256 * QB)) % N), a.N);
        if (a.obl == 0) {
          V* op = DST + (int64_t)j2 * a.R + c;
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) {
            const V w = to_v(w0, 0.f);
            pair::st16(op + kp * (256 * QB), cmul(x[P<16>(kp)], w), cmul(y[P<16>(kp)], cmul(w, wj)), pol);
            if (kp < 15) w0 = cmul(w0, st);
          }
        } else {
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) {
            const V w = to_v(w0, 0.f);
            pair::st16(DST + t1_out(a, j2, c + kp * (256 * QB)), cmul(x[P<16>(kp)], w),
                       cmul(y[P<16>(kp)], cmul(w, wj)), pol);
            if (kp < 15) w0 = cmul(w0, st);
          }
        }
      } else {
        const int kb = task * DB + dl;
        const V co = cvt(a.cout, 0.f);
        V* op = DST + (int64_t)g * 32 + 2 * cp + a.LS * (int64_t)(kb + 256 * kq);
        const int64_t step = a.LS * (int64_t)(256 * QB);
        if (a.cout.x == 1.0 && a.cout.y == 1.0) {  // forward: no conjugation, no scale
#pragma unroll
          for (int kp = 0; kp < 16; ++kp) pair::st16(op + kp * step, x[P<16>(kp)], y[P<16>(kp)], pol);
        } else {
#pragma unroll
          for (int kp = 0; kp < 16; ++kp)
            pair::st16(op + kp * step, mul2(x[P<16>(kp)], co), mul2(y[P<16>(kp)], co), pol);
        }
      }
    } else {
      // ---- A stage 1: 16-point DFTs over s -> ks, store to the ring
      //   T0 thread (pair cp = tid & 15, kt = tid >> 4): ring [kb][ja][32 lanes], kb = kt + 16 ks
      //   T1 thread (kt pair ktp = tid & 7, j2l = tid >> 3): ring [j2l][ja][ks][kt]
      const int c0 = T1 ? (tid & 7) : (tid & 15), r1 = T1 ? (tid >> 3) : (tid >> 4);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if constexpr (T1) {
          x[u] = xb[u * wide::SP + (2 * c0) * wide::KP + r1];
          y[u] = xb[u * wide::SP + (2 * c0 + 1) * wide::KP + r1];
        } else {
          const float4 t = xq[(r1 * 16 + u) * 16 + c0];
          x[u] = make_float2(t.x, t.y);
          y[u] = make_float2(t.z, t.w);
        }
      }
      reg_dft<float, 16>(x);
      reg_dft<float, 16>(y);
      const int base = T1 ? (r1 * RB + task) * 256 + 2 * c0 : (r1 * RB + task) * 32 + 2 * c0;
      const int step = T1 ? 16 : 16 * RB * 32;
      const uint64_t keep = policy_evict_last();
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) pair::st16(sp + base + ks * step, x[P<16>(ks)], y[P<16>(ks)], keep);
    }
    sc.end(a, isB, g);
  }
  sc.finish(a, nf);
#undef SRC
#undef DST
#undef STG
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// 4 CTAs per SM for both types.  (The complex128 instantiations spill 8-12
// bytes at this 128-register cap; measured at 3 CTAs per SM, ptxas spills
// 44-76 bytes instead, so 4 stays.)
template <typename R, int RA>
static void* pick_ra(int rb, bool t1) {
  constexpr int MB = 4;
  if constexpr (RA != 256) {  // the odd factor runs in the in-place pass only
    if (t1) return nullptr;
    switch (rb) {
      case 32: return (void*)lean_pass<R, RA, 32, false, MB>;
      case 64: return (void*)lean_pass<R, RA, 64, false, MB>;
      case 128: return (void*)lean_pass<R, RA, 128, false, MB>;
      case 256: return (void*)lean_pass<R, RA, 256, false, MB>;
      default: return nullptr;
    }
  } else {
    switch (rb) {
      case 32: return t1 ? (void*)lean_pass<R, RA, 32, true, MB> : (void*)lean_pass<R, RA, 32, false, MB>;
      case 64: return t1 ? (void*)lean_pass<R, RA, 64, true, MB> : (void*)lean_pass<R, RA, 64, false, MB>;
      case 128: return t1 ? (void*)lean_pass<R, RA, 128, true, MB> : (void*)lean_pass<R, RA, 128, false, MB>;
      case 256: return t1 ? (void*)lean_pass<R, RA, 256, true, MB> : (void*)lean_pass<R, RA, 256, false, MB>;
      default: return nullptr;
    }
  }
}
// 4 CTAs per SM for both types (complex64: 64 registers per thread; complex128
// tiles have half the threads but 128 registers -- a fifth CTA would spill)
template <typename R>
static void* pick(int ra, int rb, bool t1) {
  switch (ra) {
    case 192: return pick_ra<R, 192>(rb, t1);
    case 160: return pick_ra<R, 160>(rb, t1);
    case 224: return pick_ra<R, 224>(rb, t1);
    default: return pick_ra<R, 256>(rb, t1);
  }
}
template <bool PF>
static void* pick_pair_(int rb, bool t1) {
  switch (rb) {
    case 16: return t1 ? (void*)lean_pair<16, true, PF> : (void*)lean_pair<16, false, PF>;
    case 32: return t1 ? (void*)lean_pair<32, true, PF> : (void*)lean_pair<32, false, PF>;
    case 64: return t1 ? (void*)lean_pair<64, true, PF> : (void*)lean_pair<64, false, PF>;
    case 128: return t1 ? (void*)lean_pair<128, true, PF> : (void*)lean_pair<128, false, PF>;
    case 256: return t1 ? (void*)lean_pair<256, true, PF> : (void*)lean_pair<256, false, PF>;
    default: return nullptr;
  }
}
static void* pick_pair(int rb, bool t1, bool pf) { return pf ? pick_pair_<true>(rb, t1) : pick_pair_<false>(rb, t1); }
// EFFT_LEAN_PF: bit 0 = prefetching pair kernel in the transposing pass, bit 1 = in the in-place pass
static bool use_pf(bool t1) {
  const char* e = getenv("EFFT_LEAN_PF");
  const int v = e ? atoi(e) : 0;
  return (v >> (t1 ? 0 : 1)) & 1;
}
static void* pick_pipe(int rb, bool t1) {
  switch (rb) {
    case 16: return t1 ? (void*)lean_pipe<16, true> : (void*)lean_pipe<16, false>;
    case 32: return t1 ? (void*)lean_pipe<32, true> : (void*)lean_pipe<32, false>;
    case 64: return t1 ? (void*)lean_pipe<64, true> : (void*)lean_pipe<64, false>;
    case 128: return t1 ? (void*)lean_pipe<128, true> : (void*)lean_pipe<128, false>;
    case 256: return t1 ? (void*)lean_pipe<256, true> : (void*)lean_pipe<256, false>;
    default: return nullptr;
  }
}
// EFFT_LEAN_PIPE: bit 0 = the pipelined kernel in the transposing pass, bit 1 = in the in-place pass
static bool use_pipe(bool t1) {
  const char* e = getenv("EFFT_LEAN_PIPE");
  const int v = e ? atoi(e) : 0;
  return (v >> (t1 ? 0 : 1)) & 1;
}
static void* pick_wide(int rb, bool t1) {
  switch (rb) {
    case 32: return t1 ? (void*)lean_wide<32, true> : (void*)lean_wide<32, false>;
    case 64: return t1 ? (void*)lean_wide<64, true> : (void*)lean_wide<64, false>;
    case 128: return t1 ? (void*)lean_wide<128, true> : (void*)lean_wide<128, false>;
    case 256: return t1 ? (void*)lean_wide<256, true> : (void*)lean_wide<256, false>;
    default: return nullptr;
  }
}
// EFFT_LEAN_WIDE: bit 0 = the transposing pass, bit 1 = the in-place pass.
// Default 2 (measured at 2^30: in-place pass 4.93-4.94 vs 5.02-5.03 ms with the
// paired kernel; the transposing pass is 5.74 vs 5.39 ms wide, so it stays paired)
static bool use_wide(bool t1) {
  const char* e = getenv("EFFT_LEAN_WIDE");
  const int v = e ? atoi(e) : 2;
  return (v >> (t1 ? 0 : 1)) & 1;
}
static bool use_pair() {
  static const int v = getenv("EFFT_LEAN_PAIR") ? atoi(getenv("EFFT_LEAN_PAIR")) : 1;
  return v != 0;
}

// One pass: column DFTs of length R = ra * rb over `cols` columns (row
// stride cols), t1 = the transposing pass with the four-step twiddle
// W_N^((j2off + j2) k1).  Returns false when no kernel covers it.
static bool plan_pass(Pass& q, bool t1, int ra, int lb, int64_t cols, int64_t N, int64_t j2off, int c128,
                      int inverse, bool scale_inverse, bool check_finite, int num_sms, int* err_cuda,
                      bool allow_pf = true) {
  // complex64, RA = 256: the wide kernel (32-column groups, 256-byte segments)
  // when enabled and the columns divide, else the paired one (16 columns)
  const bool pipe = !c128 && ra == 256 && allow_pf && use_pipe(t1) && cols % 16 == 0;
  // (the wide kernel pays only at rho_b >= 128: measured in-place pass at 2^26 .. 2^29, rho_b 32 / 64:
  //  0.52 / 1.07 / 1.30 / 2.62 ms wide vs 0.30 / 0.58 / 1.16 / 2.32 ms paired; at 2^30, rho_b 128: 4.8-4.9 vs 5.0)
  const bool wide = !pipe && !c128 && ra == 256 && lb >= 7 && use_wide(t1) && cols % 32 == 0;
  const int F = wide ? 32 : c128 ? 8 : 16, NT = 16 * F;
  const size_t elem = c128 ? 16 : 8;
  if (cols < F || cols % F) return false;
  q.ra = ra;
  q.rb = 1 << lb;
  const int64_t R = (int64_t)ra << lb;
  const bool paired = !wide && !c128 && q.ra == 256 && use_pair();
  q.pf = paired && (pipe || use_pf(t1)) && allow_pf;  // (the sharded entries launch without tensor maps)
  q.pipe = pipe && paired;
  q.fn = reinterpret_cast<void (*)(Args)>(wide ? pick_wide(q.rb, t1)
                                          : q.pipe ? pick_pipe(q.rb, t1)
                                          : paired ? pick_pair(q.rb, t1, q.pf)
                                          : c128 ? pick<double>(q.ra, q.rb, t1) : pick<float>(q.ra, q.rb, t1));
  if (!q.fn) return false;
  q.nt = wide ? wide::NT : q.pipe ? pipe::NT : paired ? pair::NT : NT;
  q.wide = wide;
  // exchange (padded only in the transposing pass) + W_256 + W_R^(i<256) (+ two 192-entry tables)
  q.smem = wide ? (t1 ? wide::SMEM_T1 : wide::SMEM_T0)
                : q.pipe ? pipe::SMEM
                : paired ? (int)(((t1 ? pair::XB2 : 4096) + 512) * elem) + (q.pf ? 32768 : 0)
                         : (int)(((t1 ? 256 * (F + 1) : 256 * F) + 512 + (q.ra == 256 ? 0 : 2 * q.ra)) * elem);
  Args& a = q.a;
  a = Args{};
  a.R = R;
  a.N = N;
  a.j2off = j2off;
  a.LS = cols;
  a.ngroups = (int32_t)(cols / F);
  a.ntA = q.rb;
  a.ntB = wide ? q.rb : q.ra * q.rb / 256;  // wide B tiles: 64 KB as well
  a.slot_elems = (int64_t)F * R;
  a.total = (int64_t)a.ngroups * (a.ntA + a.ntB);
  a.cin = make_double2(1.0, t1 && inverse ? -1.0 : 1.0);
  const double sc = (!t1 && inverse && scale_inverse) ? 1.0 / (double)N : 1.0;
  a.cout = make_double2(sc, (!t1 && inverse) ? -sc : sc);
  a.check_finite = t1 && check_finite;
  a.abl = getenv("EFFT_PIPE_ABL") ? atoi(getenv("EFFT_PIPE_ABL")) : 0;
  if (cudaFuncSetAttribute((const void*)q.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, q.smem) != cudaSuccess) {
    *err_cuda = 1;
    return false;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)q.fn, q.nt, q.smem) != cudaSuccess ||
      occ < 1) {
    *err_cuda = 1;
    return false;
  }
  q.grid = occ * num_sms;
  // Claimed tasks in flight span about 3 grids: B(g) is issued `lag` groups
  // after A(g), and A(g) reuses the slot of group g - nslots.
  // W adjacent groups interleaved (decode); lag in super-groups of W, slots in groups
  int64_t W = 1;
  if (const char* ev = getenv("EFFT_LEAN_W")) W = atoi(ev);
  while (W > 1 && a.ngroups % W) W /= 2;
  if (W < 1) W = 1;
  a.wg = (int32_t)W;
  const int64_t G = a.ngroups / W;
  const int64_t per = ((int64_t)a.ntA + a.ntB) * W;
  // (pipelined kernel, static schedule: three groups per CTA, two tiles each in flight, the next one probed)
  const int64_t window = ((q.pipe ? 9 : 4) * (int64_t)q.grid + per - 1) / per;
  // (measured at 2^30: paired 10:16 4.97 / 4.77 ms vs 11:18 5.06 / 4.89 and 13:20 5.44 / 5.13;
  //  wide in-place pass 5:8 4.62 ms vs 6:9 4.69 and 8:12 5.16 -- the ring must stay well inside L2)
  // (pipelined kernel: a finished tile is published ~2 tile periods late -- lag 8, 14 slots at 2^30)
  int64_t lag = window + (getenv("EFFT_LEAN_LAGPLUS") ? atoi(getenv("EFFT_LEAN_LAGPLUS")) : q.pipe ? 2 : 0);
  if (const char* ev = getenv("EFFT_LEAN_LAG")) lag = atoi(ev);
  int64_t slots = wide ? lag + 3 : q.pipe ? lag + window : lag + (window + 1) / 2 + 1;  // super-groups (wide: 8 MB slots)
  if (const char* ev = getenv("EFFT_LEAN_SLOTS")) slots = atoi(ev);
  if (lag < 1) lag = 1;
  if (lag > G) lag = G;
  if (slots < lag + 1) slots = lag + 1;
  if (slots > G) slots = G;
  a.lag = (int32_t)lag;
  a.nslots = (int32_t)(slots * W);
  q.counter_ints = 2 + 2 * (int64_t)a.ngroups;
  return true;
}

static bool factor_m(int64_t n, int& m, int& t) {
  if (n <= 0) return false;
  int64_t mm = n;
  t = 0;
  while ((mm & 1) == 0) {
    mm >>= 1;
    ++t;
  }
  m = (int)mm;
  return m == 1 || m == 3 || m == 5 || m == 7;
}

// in-place pass: RA2 = 256, or 12 x 16 = 3 * 64, 10 x 16 = 5 * 32, 14 x 16 = 7 * 32
static int ra_of(int m) { return m == 3 ? 192 : m == 5 ? 160 : m == 7 ? 224 : 256; }
// log2(RB) of an R = ra * 2^lb pass; rho_b >= 32 (QB >= 2) in general, the
// paired complex64 kernel also runs rho_b = 16 (QB = 1)
static bool rb_ok(int lb, int c128, int m) { return lb >= ((!c128 && m == 1) ? 4 : 5) && lb <= 8; }

bool plan(int64_t n, int c128, int inverse, bool scale_inverse, bool check_finite, int num_sms, Pass p[2],
          int64_t* staging_elems, int* err_cuda) {
  *err_cuda = 0;
  int m, t;
  if (!factor_m(n, m, t)) return false;
  // RA = 256, except RA = 192 / 160 / 224 in pass 2 (the in-place pass) when 3 / 5 / 7 | n
  const int ra2 = ra_of(m);
  const int lbs = m == 1 ? t - 16 : m == 3 ? t - 14 : t - 13;
  const int lb1 = (lbs + 1) / 2, lb2 = lbs - lb1;
  if (!rb_ok(lb1, c128, m) || !rb_ok(lb2, c128, m)) return false;
  const int64_t R1 = int64_t(256) << lb1, R2 = (int64_t)ra2 << lb2;
  if (!plan_pass(p[0], true, 256, lb1, R2, n, 0, c128, inverse, scale_inverse, check_finite, num_sms, err_cuda) ||
      !plan_pass(p[1], false, ra2, lb2, R1, n, 0, c128, inverse, scale_inverse, check_finite, num_sms, err_cuda))
    return false;
  *staging_elems = std::max(p[0].a.nslots * p[0].a.slot_elems, p[1].a.nslots * p[1].a.slot_elems);
  return true;
}

int lanes(int c128) { return c128 ? 8 : 32; }

bool split_sharded(int64_t n, int G, int c128, int64_t* N1, int64_t* N2) {
  int m, t;
  if (!factor_m(n, m, t) || G < 1 || (G & (G - 1))) return false;
  const int ra2 = ra_of(m);
  const int lbs = m == 1 ? t - 16 : m == 3 ? t - 14 : t - 13;
  const int lb1 = (lbs + 1) / 2, lb2 = lbs - lb1;
  if (!rb_ok(lb1, c128, m) || !rb_ok(lb2, c128, m)) return false;
  *N1 = int64_t(256) << lb1;
  *N2 = (int64_t)ra2 << lb2;
  const int F = c128 ? 8 : 16;
  return *N1 % ((int64_t)G * F) == 0 && *N2 % ((int64_t)G * F) == 0;
}

bool plan_sharded(int64_t n, int G, int rank, int c128, int inverse, bool check_finite, int num_sms, Pass p[2],
                  int64_t* staging_elems, int* err_cuda, bool blocked, int chunks) {
  *err_cuda = 0;
  int64_t N1, N2;
  if (!split_sharded(n, G, c128, &N1, &N2)) return false;
  int m, t;
  factor_m(n, m, t);
  const int ra2 = ra_of(m);
  int lb1 = 0, lb2 = 0;
  while ((int64_t(256) << lb1) < N1) ++lb1;
  while (((int64_t)ra2 << lb2) < N2) ++lb2;
  const int64_t L1 = N1 / G, L2 = N2 / G;
  // pass 1 over this rank's L2 columns (global columns rank * L2 + c), pass 2 over its L1 columns;
  // chunks > 1 (the overlapped single-process entry): each launch covers 1 / chunks of the
  // columns -- the row strides stay L2 and L1, the launcher offsets src / dst / j2off
  if (chunks < 1 || L2 % chunks || L1 % chunks) return false;
  if (!plan_pass(p[0], true, 256, lb1, L2 / chunks, n, (int64_t)rank * L2, c128, inverse, true, check_finite,
                 num_sms, err_cuda, false) ||
      !plan_pass(p[1], false, ra2, lb2, L1 / chunks, n, 0, c128, inverse, true, check_finite, num_sms, err_cuda,
                 false))
    return false;
  p[0].a.LS = L2;
  p[1].a.LS = L1;
  if (blocked) {
    int lg = 0;
    while ((int64_t(1) << lg) < L1) ++lg;
    if ((int64_t(1) << lg) != L1 || L1 < 2) return false;
    p[0].a.obl = lg;
  }
  *staging_elems = std::max(p[0].a.nslots * p[0].a.slot_elems, p[1].a.nslots * p[1].a.slot_elems);
  return true;
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

int encode_input(Pass& p, const void* src) {
  EncodeTiledFn enc = encoder();
  if (!enc) return 1;
  Args& a = p.a;
  const int64_t RB = p.rb;
  cuuint64_t dims[3] = {(cuuint64_t)a.LS, (cuuint64_t)RB, 256};
  cuuint64_t strides[2] = {(cuuint64_t)(a.LS * 8), (cuuint64_t)(RB * a.LS * 8)};
  cuuint32_t box[3] = {16, 1, 256};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&a.mapA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(src), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return (int)r;
  p.mapA_ptr = src;
  return 0;
}

int encode_ring(Pass& p, void* staging) {
  EncodeTiledFn enc = encoder();
  if (!enc) return 1;
  Args& a = p.a;
  const int64_t RB = p.rb, DB = 256 / RB;
  // T1 ring [j2l 16][ja RB][ks 16][kt 16] per slot
  cuuint64_t dims[5] = {16, 16, (cuuint64_t)RB, 16, (cuuint64_t)a.nslots};
  cuuint64_t strides[4] = {16 * 8, 256 * 8, (cuuint64_t)(RB * 256 * 8), (cuuint64_t)(16 * RB * 256 * 8)};
  cuuint32_t box[5] = {16, 1, (cuuint32_t)RB, (cuuint32_t)DB, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&a.mapB, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, staging, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace lean
}  // namespace efft

// tpass.cu -- TMA-pipelined, warp-specialised staged passes for complex64,
// N = 2^30 (configuration C3).
//
// The algorithm is the four-step form of the reference's scatter -> leaves ->
// merges (scatter.py:31-57, leaf_dft.py:93-125, recombine.py:144-260), as in
// lean.cu; what changes is how a pass meets the memory system (tpass.cuh).
//
// Index maps (per pass: R = RA RB, RA = 256, RB = 128; F = 32 columns):
//   column DFT point j = ja + RB jb, output k = ka + RA kb;
//   A tile (group g, residue ja): 256 jb x 32 columns from HBM (one TMA box),
//     256-point DFT over jb (16 x 16: jb = s + 16 t, ka = kt + 16 ks), times
//     W_R^(ja ka), to the group's L2 staging slot;
//   B tile: 128-point DFT over ja (8 x 16: ja = p + 16 q, kb = kq + 8 kp) of
//     64 (ka, column) lines from the slot (one TMA box / bulk copy), to HBM.
//   pass 1 (T1): x[j2 + R2 j1] -> y[k1 + R1 j2] W_N^(j2 k1), columns j2;
//                slot layout [column][ja][ka]; B tile = one column, 64 ka
//   pass 2 (T0): y[k1 + R1 j2] -> X[k1 + R1 k2] in place, columns k1;
//                slot layout [ka][ja][column]; B tile = two ka, 32 columns
//
// One CTA per SM (measured: tools/skel_bench.cu, profiles/):
//   * warp 16 is the producer: claims tasks from the pass counter, waits for a
//     task's producers (B(g): all A(g) tiles released; A(g): the slot's
//     previous group consumed), issues the tile's TMA into one of three 64 KB
//     landing buffers, computes the tile's twiddles in fp64 from exact integer
//     exponents, and releases finished tiles (fence.acq_rel + add) -- none of
//     which ever stalls the compute warps;
//   * warps 0-15 are two independent compute groups of 256 threads; each owns
//     half of every tile (16 values per thread), exchanges between its two
//     radix stages IN PLACE in the landing buffer (XOR-swizzled rows, no bank
//     conflicts) behind its own named barrier, and hands the buffer back
//     through an mbarrier as soon as its last shared-memory read is done.
// Deadlock freedom: tasks are claimed in one global order whose dependencies
// all point backwards; the producer services releases while it waits, and the
// compute groups never wait on anything but tiles already being loaded.
#include <cstdlib>

#include "efft_kernels.cuh"
#include "tpass.cuh"

namespace efft {
namespace tpass {

constexpr int NCW = 16;          // compute warps (two groups of 8)
constexpr int NT = NCW * 32 + 64;  // + the producer and helper warps
constexpr int F = 32;            // columns per group (256-byte segments)
constexpr int RA = 256;
constexpr int RB = 128;
constexpr int TILE = 8192;       // elements per tile (64 KB)
constexpr int NBUF = 3;          // landing buffers
constexpr int NTW = 256;         // per-tile twiddles (float2)
constexpr int SMEM = NBUF * TILE * 8 + 256 * 16 + 4 * NTW * 16;

template <int S>
__device__ __forceinline__ constexpr int P(int k) {
  return dif_pos_t<S>(k);
}

__device__ __forceinline__ float2 f2(double2 w) { return make_float2((float)w.x, (float)w.y); }
// twiddles are kept as (re, im, -im, re): a complex multiply is then FMUL2 + FFMA2
__device__ __forceinline__ float4 f4(double2 w) {
  const float x = (float)w.x, y = (float)w.y;
  return make_float4(x, y, -y, x);
}
__device__ __forceinline__ float2 cm4(float2 v, float4 w) {
  return fma2(make_float2(v.y, v.y), make_float2(w.z, w.w), mul2(make_float2(v.x, v.x), make_float2(w.x, w.y)));
}
// (a w) for a pair of float4 twiddles, kept in float4 form
__device__ __forceinline__ float4 cm44(float4 a, float4 w) {
  const float2 r = cm4(make_float2(a.x, a.y), w);
  return make_float4(r.x, r.y, -r.y, r.x);
}

// weak 8-byte store with an L2 eviction-policy hint (st.global.cg would make it a
// strong GPU-scope store; ordering comes from the mbarrier / fence release instead)
__device__ __forceinline__ void st8(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
               : "memory");
}

// Position -> (isB, group, task) of the claim order (see lean.cu).
__device__ __forceinline__ void decode(const Args& a, uint32_t pos, int& isB, int& g, int& task) {
  const uint32_t L = a.lag, na = a.ntA, nb = a.ntB, per = na + nb, G = a.ngroups;
  if (pos < L * na) {
    isB = 0;
    g = (int)(pos / na);
    task = (int)(pos % na);
  } else if (pos < L * na + (G - L) * per) {
    const uint32_t q = pos - L * na;
    const uint32_t i = L + q / per, r = q % per;
    isB = r < nb;
    g = (int)(isB ? i - L : i);
    task = (int)(isB ? r : r - nb);
  } else {
    const uint32_t q = pos - L * na - (G - L) * per;
    isB = 1;
    g = (int)(G - L + q / nb);
    task = (int)(q % nb);
  }
}

struct Task {
  int valid, isB, g, task;
};

// bounded mbarrier wait: a lost completion traps instead of hanging the GPU
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity, int tag) {
  long long n = 0;
  while (!mbar_try(bar, parity)) {
    if (++n == (1ll << 26)) {
      printf("EFFT tpass: barrier %d never completed cta=%d thread=%d\n", tag, blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

__device__ __forceinline__ void named_bar(int id) {
  asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}
#define NAMED_BAR(id)                          \
  do {                                         \
    const long long tb_ = prof ? clock64() : 0; \
    named_bar(id);                             \
    if (prof) cbar += clock64() - tb_;         \
  } while (0)

// ---------------------------------------------------------------- producer (one lane)
// diagnostics (a.prof, EFFT_TP_PROF): cycle sums over CTAs, added into a.prof at exit
//   [0] producer dependency waits  [1] producer buffer waits  [2] producer total
//   [3] compute wait for tiles (warp 0)  [4] compute barrier waits (warp 0)  [5] compute total (warp 0)
//   [6] helper twiddle cycles  [7] tiles
constexpr int NTS = 4;  // task-info / twiddle slots: tile k's are reused by tile k+4, issued only
                        // after every warp read tile k+1, i.e. after tile k was finished

// per-tile twiddles in fp64, rounded once (all 32 helper lanes)
//   A tile:    tw[ka] = W_R^(ja ka), ka < 256 (the W_R^(ja kt) W_R^(16 ja ks) product in fp64)
//   T1 B tile: tw[i] = W_N^(j2 (64 kab + i)), i < 64; tw[64 + kb] = W_N^(256 j2 kb), kb < 128
template <bool T1>
__device__ __forceinline__ void tile_twiddles(const Args& a, const Task& t, float4* tw, int lane) {
  if (!t.isB) {
    const int64_t R = a.R, ja = t.task;
    const double2 lo = wroot((ja * (lane & 15)) % R, R);           // W_R^(ja kt), kt = lane & 15
    const double2 hi0 = wroot((16 * ja * (lane >> 4)) % R, R);     // W_R^(16 ja ks), ks = lane >> 4
    const double2 st = wroot((32 * ja) % R, R);                    // W_R^(32 ja): ks += 2
    double2 h = hi0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {  // ka = (lane & 15) + 16 (2 m + (lane >> 4))
      const double2 w = make_double2(lo.x * h.x - lo.y * h.y, lo.x * h.y + lo.y * h.x);
      tw[(lane & 15) + 16 * (2 * m + (lane >> 4))] = f4(w);
      h = make_double2(h.x * st.x - h.y * st.y, h.x * st.y + h.y * st.x);
    }
  } else if (T1) {
    const int64_t N = a.N, j2 = (int64_t)t.g * F + (t.task >> 2), kab = t.task & 3;
    double2 w[6];
#pragma unroll
    for (int m = 0; m < 6; ++m) {  // independent: the six sincospi overlap
      const int i = lane + 32 * m;
      const int64_t e = i < 64 ? j2 * (64 * kab + i) : (int64_t)256 * j2 * (i - 64);
      w[m] = wroot(e % N, N);
    }
#pragma unroll
    for (int m = 0; m < 6; ++m) tw[lane + 32 * m] = f4(w[m]);
  }
}

template <bool T1, bool PROF>
__global__ void __launch_bounds__(NT, 1) tpass128(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* const land0 = reinterpret_cast<float2*>(smraw);
  float4* const w256 = reinterpret_cast<float4*>(smraw + NBUF * TILE * 8);
  float4* const twb = w256 + 256;  // [NTS][NTW]
  __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF], stored[NBUF], info[NTS];
  __shared__ Task task_sh[NTS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < 256; i += NT) w256[i] = f4(wroot(i, 256));
  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full[b], 2);  // producer (expect_tx) + helper (task twiddles ready)
      mbar_init(&empty[b], NCW);
      mbar_init(&stored[b], NCW);
    }
    for (int i = 0; i < NTS; ++i) mbar_init(&info[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long tstart = clock64();

  if (warp == NCW) {
    // ======================================================== producer warp (lane 0)
    // The next task is claimed and its producers checked while the compute
    // warps work through the tiles already loaded; when a landing buffer
    // frees, its TMA goes out at once.
    if (lane != 0) return;
    unsigned long long wdep = 0, wslot = 0;
    auto claim = [&](Task& t) {
      const unsigned long long pos = atomicAdd(a.ctr, 1ull);
      t.valid = pos < (unsigned long long)a.total;
      t.isB = t.g = t.task = 0;
      if (!t.valid) return;
      decode(a, (uint32_t)pos, t.isB, t.g, t.task);
      const int32_t* c = t.isB ? a.doneA + t.g : (t.g >= a.nslots ? a.doneB + (t.g - a.nslots) : nullptr);
      const int32_t need = t.isB ? a.ntA : a.ntB;
      if (c && ld_acquire(c) < need) {  // rare: wait (the helper warp keeps releasing meanwhile)
        const long long t0 = clock64();
        long long n = 0;
        while (ld_acquire(c) < need) {
          __nanosleep(64);
          if (++n == (1ll << 26)) {
            printf("EFFT tpass stuck cta=%d need=%d have=%d\n", blockIdx.x, need, ld_acquire(c));
            __trap();
          }
        }
        wdep += clock64() - t0;
      }
    };
    Task t;
    claim(t);
    for (long long k = 0;; ++k) {
      const int b = (int)(k % NBUF), ts = (int)(k % NTS);
      if (k >= NBUF) {
        const long long t0 = clock64();
        wait_bar(&empty[b], (uint32_t)((k / NBUF - 1) & 1), 1);
        wslot += clock64() - t0;
      }
      // (slot ts held tile k-4: empty(k-3) above means every compute warp finished
      // tile k-4 and the helper, which arrived on full(k-3), consumed its info)
      task_sh[ts] = t;
      if (!t.valid) {
        mbar_arrive(&full[b]);  // terminator: the helper adds the second arrival
        mbar_arrive(&info[ts]);
        break;
      }
      // ring stores observed through the acquire, before the async-proxy read
      asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_arrive_tx(&full[b], TILE * 8);
      const uint64_t pol = policy_evict_first();  // HBM input and ring lines are read once
      float2* land = land0 + (size_t)b * TILE;
      const int slot = t.g % a.nslots;
      if (!t.isB) {
        tma_load_3d(land, &a.mapA, t.g * F, t.task, 0, &full[b], pol);
      } else if constexpr (T1) {
        tma_load_4d(land, &a.mapB, 64 * (t.task & 3), 0, t.task >> 2, slot, &full[b], pol);
      } else {
        const float2* src = reinterpret_cast<const float2*>(a.stg) + (int64_t)slot * a.slot_elems +
                            (int64_t)(2 * t.task) * RB * F;
        bulk_g2s(land, src, TILE * 8, &full[b], pol);
      }
      mbar_arrive(&info[ts]);  // release: task info for the helper and the compute warps
      claim(t);
    }
    if (PROF) {
      atomicAdd(a.prof + 0, wdep);
      atomicAdd(a.prof + 1, wslot);
      atomicAdd(a.prof + 2, (unsigned long long)(clock64() - tstart));
    }
    return;
  }
  if (warp == NCW + 1) {
    // ======================================================== helper warp
    // per-tile twiddles, then the release of finished tiles (fence.acq_rel +
    // add, in tile order, one fence for all tiles found finished)
    int32_t* done_ring[8];  // at most 6 tiles are unreleased when a new one is published
    long long released = 0, k = 0;
    unsigned long long twc = 0;
    auto service = [&]() {
      if (lane != 0) return;
      int n = 0;
      int32_t* ptrs[NBUF];
      while (released < k && n < NBUF) {
        if (!mbar_try(&stored[released % NBUF], (uint32_t)((released / NBUF) & 1))) break;
        ptrs[n++] = done_ring[released & 7];
        ++released;
      }
      if (n) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int i = 0; i < n; ++i) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(ptrs[i]) : "memory");
      }
    };
    for (;; ++k) {
      const int ts = (int)(k % NTS);
      long long n = 0;
      while (true) {  // wait for the task info, releasing finished tiles meanwhile
        int ok = lane == 0 ? mbar_try(&info[ts], (uint32_t)((k / NTS) & 1)) : 0;
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (ok) break;
        service();
        if (++n == (1ll << 28)) __trap();
      }
      const Task t = task_sh[ts];
      if (!t.valid) {
        if (lane == 0) mbar_arrive(&full[k % NBUF]);
        break;
      }
      const long long t0 = clock64();
      tile_twiddles<T1>(a, t, twb + ts * NTW, lane);
      twc += clock64() - t0;
      if (lane == 0) done_ring[k & 7] = t.isB ? a.doneB + t.g : a.doneA + t.g;
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[k % NBUF]);  // release: twiddles visible with the tile
      service();
    }
    if (lane == 0) {
      long long n = 0;
      while (released < k) {
        service();
        if (++n == (1ll << 28)) __trap();
      }
      if (PROF) {
        atomicAdd(a.prof + 6, twc);
        atomicAdd(a.prof + 7, (unsigned long long)k);
      }
    }
    return;
  }

  // ========================================================== compute groups
  const int gid = warp >> 3;       // group: half of every tile
  const int lw = warp & 7;         // warp within the group
  const int bar_id = 1 + gid;
  const uint64_t pol_out = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  float2* const STG = reinterpret_cast<float2*>(a.stg);
  float2* const DST = reinterpret_cast<float2*>(a.dst);
  bool nf = false;
  unsigned long long cwait = 0, cbar = 0;
  const bool prof = PROF && tid == 0;
  unsigned long long ph[2][6] = {};  // [A/B][ld, st0, bar+sts+bar, ld1, st1+stores, end]
  long long tl = 0;
#define PH(kind, i)                          \
  do {                                       \
    if (prof) {                              \
      const long long n_ = clock64();        \
      ph[kind][i] += (unsigned long long)(n_ - tl); \
      tl = n_;                               \
    }                                        \
  } while (0)

  // The "stores of tile k done" arrival (release) waits for the warp's stores
  // to drain; it is deferred to after tile k+1's shared loads, when they have.
  // If tile k+1 is not loaded yet -- its producers may include tile k -- the
  // arrival is made at once (no waiting while holding an unreleased tile).
  int pend_st = -1;
  auto arrive_stored = [&]() {
    if (pend_st >= 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&stored[pend_st]);
      pend_st = -1;
    }
  };
  for (long long k = 0;; ++k) {
    const int b = (int)(k % NBUF);
    long long tp0 = prof ? clock64() : 0;
    if (pend_st >= 0) {
      int ok = lane == 0 ? mbar_try(&full[b], (uint32_t)((k / NBUF) & 1)) : 0;
      if (!__shfl_sync(0xffffffffu, ok, 0)) arrive_stored();
    }
    wait_bar(&full[b], (uint32_t)((k / NBUF) & 1), 0);
    if (prof) {
      cwait += clock64() - tp0;
      tl = clock64();
    }
    const Task t = task_sh[k % NTS];
    if (!t.valid) {
      arrive_stored();
      break;
    }
    float2* const L = land0 + (size_t)b * TILE;
    const float4* const tw = twb + (k % NTS) * NTW;
    float2* const sp = STG + (int64_t)(t.g % a.nslots) * a.slot_elems;
    float2 v[16];

    if (!t.isB) {
      // ================= A tile: columns 16 gid + c, 256-point DFTs over jb = s + 16 t
      const int c = lane & 15, s = 2 * lw + (lane >> 4);
      const int col = 16 * gid + c;
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = L[(16 * u + s) * F + col];
      if (T1 && a.check_finite) {
#pragma unroll
        for (int u = 0; u < 16; ++u) nf |= !(isfinite(v[u].x) && isfinite(v[u].y));
      }
      if constexpr (T1) {
        const float2 ci = f2(a.cin);
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = mul2(v[u], ci);
      }
      arrive_stored();
      PH(0, 0);
      reg_dft<float, 16>(v);
#pragma unroll
      for (int kk = 1; kk < 16; ++kk) v[P<16>(kk)] = cm4(v[P<16>(kk)], w256[s * kk]);
      PH(0, 1);
      NAMED_BAR(bar_id);  // the group's half of the landing buffer is read
      // in place: value (kt, s) -> row 16 kt + s, column 16 gid + (c ^ kt); the row
      // base is a multiple of 128 bytes, so the address is (base ^ 8 kt) + 4096 kt
      {
        const uint32_t a0 = smem_u32(L) + (uint32_t)(s * 256 + gid * 128 + c * 8);
#pragma unroll
        for (int kt = 0; kt < 16; ++kt) {
          const float2 x = v[P<16>(kt)];
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"((a0 ^ (uint32_t)(8 * kt)) + 4096u * kt), "f"(x.x), "f"(x.y)
                       : "memory");
        }
      }
      NAMED_BAR(bar_id);
      int kt, cc;
      if constexpr (T1) {  // lanes: 16 kt x 2 columns (ring rows of 16 consecutive ka)
        kt = lane & 15;
        cc = 2 * lw + (lane >> 4);
      } else {  // lanes: 16 columns x 2 kt (ring rows of 16 consecutive columns)
        cc = lane & 15;
        kt = 2 * lw + (lane >> 4);
      }
      PH(0, 2);
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = L[(16 * kt + u) * F + 16 * gid + (cc ^ kt)];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
      PH(0, 3);
      reg_dft<float, 16>(v);
      if constexpr (T1) {  // ring [column][ja][ka], ka = kt + 16 ks
        float2* op = sp + ((int64_t)(16 * gid + cc) * RB + t.task) * 256 + kt;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) st8(op + 16 * ks, cm4(v[P<16>(ks)], tw[kt + 16 * ks]), pol_keep);
      } else {  // ring [ka][ja][column]
        float2* op = sp + ((int64_t)kt * RB + t.task) * F + 16 * gid + cc;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks)
          st8(op + (int64_t)16 * ks * RB * F, cm4(v[P<16>(ks)], tw[kt + 16 * ks]), pol_keep);
      }
    } else {
      // ================= B tile: 128-point DFTs over ja = p + 16 q, kb = kq + 8 kp
      // T1: landing [ja][64 ka], group half = ka 32 gid + (0..31), lines = ka
      // T0: landing [kal][ja][32 col], group = kal, lines = columns
      const int ln = lane, pp = lw;  // stage 0: line, p in {pp, pp + 8}
      const int rowbase = T1 ? 0 : gid * RB;
      const int pitch = T1 ? 64 : F;
      const int lc = T1 ? 32 * gid + ln : ln;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = L[(rowbase + pp + 16 * q) * pitch + lc];
        v[8 + q] = L[(rowbase + pp + 8 + 16 * q) * pitch + lc];
      }
      {  // the consumed ring lines leave L2 without write-back (one line per thread and group)
        const float2* rp = T1 ? sp + ((int64_t)(t.task >> 2) * RB) * 256 + 64 * (t.task & 3)
                              : sp + (int64_t)(2 * t.task) * RB * F;
        const int i = lw * 32 + lane;  // 256 lines per group half
        if constexpr (T1) {
          if (i < 256) l2_discard(rp + (i >> 1) * 256 + 32 * gid + (i & 1) * 16);
        } else {
          l2_discard(rp + (int64_t)gid * RB * F + i * 16);
        }
      }
      arrive_stored();
      PH(1, 0);
      reg_dft<float, 8>(v);
      reg_dft<float, 8>(v + 8);
#pragma unroll
      for (int kk = 1; kk < 8; ++kk) {  // W_128^(p kq) = W_256^(2 p kq)
        v[P<8>(kk)] = cm4(v[P<8>(kk)], w256[2 * pp * kk]);
        v[8 + P<8>(kk)] = cm4(v[8 + P<8>(kk)], w256[2 * (pp + 8) * kk]);
      }
      PH(1, 1);
      NAMED_BAR(bar_id);
      // in place: value (kq, p) of line ln -> row 16 kq + p
#pragma unroll
      for (int kq = 0; kq < 8; ++kq) {
        L[(rowbase + 16 * kq + pp) * pitch + lc] = v[P<8>(kq)];
        L[(rowbase + 16 * kq + pp + 8) * pitch + lc] = v[8 + P<8>(kq)];
      }
      NAMED_BAR(bar_id);
      PH(1, 2);
      const int kq = lw;  // stage 1: line, kq
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = L[(rowbase + 16 * kq + u) * pitch + lc];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
      PH(1, 3);
      reg_dft<float, 16>(v);
      if constexpr (T1) {
        // y[k1 + R1 j2] = Y W_N^(j2 k1), k1 = ka + 256 (kq + 8 kp), ka = 64 kab + 32 gid + ln
        const int j2 = t.g * F + (t.task >> 2), kab = t.task & 3;
        const float4 a0 = tw[32 * gid + ln];
        float2* op = DST + (int64_t)j2 * a.R + 64 * kab + 32 * gid + ln + 256 * kq;
#pragma unroll
        for (int kp = 0; kp < 16; ++kp) st8(op + 2048 * kp, cm4(v[P<16>(kp)], cm44(a0, tw[64 + kq + 8 * kp])), pol_out);
      } else {
        // X[k1 + R1 k2], k2 = ka + 256 (kq + 8 kp), ka = 2 task + gid, k1 = 32 g + ln
        const float2 co = f2(a.cout);
        const int ka = 2 * t.task + gid;
        float2* op = DST + (int64_t)(ka + 256 * kq) * a.LS + t.g * F + ln;
        const int64_t step = (int64_t)2048 * a.LS;
#pragma unroll
        for (int kp = 0; kp < 16; ++kp) st8(op + kp * step, mul2(v[P<16>(kp)], co), pol_out);
      }
    }
    PH(t.isB, 4);
    pend_st = b;  // release (cta) of this warp's stores of the tile, deferred
    PH(t.isB, 5);
  }
  if (nf) atomicOr(a.flag, 1);
  if (prof) {
    for (int i = 0; i < 12; ++i) atomicAdd(a.prof + 8 + i, ph[i / 6][i % 6]);
    atomicAdd(a.prof + 3, cwait);
    atomicAdd(a.prof + 4, cbar);
    atomicAdd(a.prof + 5, (unsigned long long)(clock64() - tstart));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
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

static bool env_on(const char* k, int dflt) {
  const char* v = getenv(k);
  return v ? atoi(v) != 0 : dflt != 0;
}

bool plan(int64_t n, int c128, int inverse, bool check_finite, int num_sms, Pass p[2], int64_t* staging_elems,
          int* err_cuda) {
  *err_cuda = 0;
  if (c128 || n != (int64_t(1) << 30) || !env_on("EFFT_TPASS", 0) || !encoder()) return false;
  const int64_t R1 = int64_t(1) << 15, R2 = int64_t(1) << 15;
  int64_t stg = 0;
  for (int i = 0; i < 2; ++i) {
    Pass& q = p[i];
    const bool t1 = i == 0;
    q = Pass{};
    q.rb = 128;
    q.fn = reinterpret_cast<void (*)(Args)>(t1 ? tpass128<true, false> : tpass128<false, false>);
    q.fn_prof = reinterpret_cast<void (*)(Args)>(t1 ? tpass128<true, true> : tpass128<false, true>);
    q.nt = NT;
    q.smem = SMEM;
    Args& a = q.a;
    a.R = t1 ? R1 : R2;
    a.N = n;
    a.LS = t1 ? R2 : R1;
    a.ngroups = (int32_t)((t1 ? R2 : R1) / F);
    a.ntA = 128;
    a.ntB = 128;
    a.slot_elems = (int64_t)F * a.R;
    a.total = (int64_t)a.ngroups * (a.ntA + a.ntB);
    a.cin = make_double2(1.0, t1 && inverse ? -1.0 : 1.0);
    const double sc = (!t1 && inverse) ? 1.0 / (double)n : 1.0;
    a.cout = make_double2(sc, (!t1 && inverse) ? -sc : sc);
    a.check_finite = t1 && check_finite;
    if (cudaFuncSetAttribute((const void*)q.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, q.smem) != cudaSuccess ||
        cudaFuncSetAttribute((const void*)q.fn_prof, cudaFuncAttributeMaxDynamicSharedMemorySize, q.smem) !=
            cudaSuccess) {
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
    // tasks in flight: up to NBUF per CTA
    const int64_t per = (int64_t)a.ntA + a.ntB;
    const int64_t window = (NBUF * (int64_t)q.grid + per - 1) / per;
    // measured (tools/tp_check.py, lag/slot sweep at 2^30): lag 6 / 9 slots of 8 MB
    int64_t lag = 3 * window;
    if (const char* ev = getenv("EFFT_TP_LAG")) lag = atoi(ev);
    int64_t slots = lag + window + 1;
    if (const char* ev = getenv("EFFT_TP_SLOTS")) slots = atoi(ev);
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

int encode_input(Pass& p, int pass_index, const void* src) {
  EncodeTiledFn enc = encoder();
  if (!enc) return 1;
  const Args& a = p.a;
  const int64_t RB = a.R / RA;
  cuuint64_t dims[3] = {(cuuint64_t)a.LS, (cuuint64_t)RB, (cuuint64_t)RA};
  cuuint64_t strides[2] = {(cuuint64_t)(a.LS * 8), (cuuint64_t)(RB * a.LS * 8)};
  cuuint32_t box[3] = {(cuuint32_t)F, 1, (cuuint32_t)RA};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&p.a.mapA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(src), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  (void)pass_index;
  if (r != CUDA_SUCCESS) return (int)r;
  p.mapA_ptr = src;
  return 0;
}

int encode_ring(Pass& p, void* staging) {
  EncodeTiledFn enc = encoder();
  if (!enc) return 1;
  const int64_t RB = p.a.R / RA;
  cuuint64_t dims[4] = {256, (cuuint64_t)RB, (cuuint64_t)F, (cuuint64_t)p.a.nslots};
  cuuint64_t strides[3] = {256 * 8, (cuuint64_t)(RB * 256 * 8), (cuuint64_t)(F * RB * 256 * 8)};
  cuuint32_t box[4] = {64, (cuuint32_t)RB, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&p.a.mapB, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, staging, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace tpass
}  // namespace efft

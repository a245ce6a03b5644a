// efft_kernels.cuh -- sm_100a kernels for one very large 1D complex DFT.
//
// A transform of N = M * 2^t (M in {1, 3}) runs as at most two Stockham
// "passes" (N = R1 * R2), each one HBM read + one HBM write of the array.  A
// pass does R-point DFTs down the columns of an (R x N/R) view with the
// decimation-in-time twiddle of the pass fused into the load and the Stockham
// transpose fused into the store.  This is the four-step decomposition that the
// reference's scatter / leaf / merge stages compute on the CPU:
//   scatter  (reference scatter.py:31-57)       -> the strided column load of pass 1
//   leaves   (reference leaf_dft.py:93-125)     -> the column DFTs of the passes
//   merges   (reference recombine.py:144-260)   -> twiddles W_N^(k*r) + the pass-2 DFTs
//
// When R is larger than one CTA can hold, the pass is "staged": R = rho_a *
// rho_b, sub-stage A does rho_a-point DFTs from HBM into an L2-resident staging
// ring, sub-stage B does rho_b-point DFTs from the ring to HBM.  Both task
// types run in ONE persistent kernel; B tasks of a column group wait on a
// per-group counter for its A tasks, so the staging traffic stays in L2 and
// each pass still costs one HBM read and one HBM write.
//
// A task ("tile") is F x D x RHO complex elements: F adjacent columns (F *
// sizeof(complex) = 128 B, so every global access is a full 128-byte line and
// every shared-memory row touches all 32 banks exactly once), D independent
// DFTs, RHO points each.  The tile lives in registers (E elements per thread)
// and is exchanged through padded shared memory between in-CTA radix stages.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "w192_table.cuh"

namespace efft {

// ----------------------------------------------------------------------------
// complex helpers
// ----------------------------------------------------------------------------
template <typename R> struct CT;
template <> struct CT<float> {
  using V = float2;
  static constexpr int F = 16;
};
template <> struct CT<double> {
  using V = double2;
  static constexpr int F = 8;
};

__device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return mk(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return mk(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 to_v(double2 w, float) { return make_float2((float)w.x, (float)w.y); }
__device__ __forceinline__ double2 to_v(double2 w, double) { return w; }

template <typename R> __device__ __forceinline__ typename CT<R>::V w192(int q);
template <> __device__ __forceinline__ float2 w192<float>(int q) {
  return make_float2(c_w192_float[q][0], c_w192_float[q][1]);
}
template <> __device__ __forceinline__ double2 w192<double>(int q) {
  return make_double2(c_w192_double[q][0], c_w192_double[q][1]);
}

// b * W_N^k with N | 192; k, N are compile-time after unrolling so the branches
// fold and the table read becomes a constant-bank operand.
template <typename R, int N>
__device__ __forceinline__ typename CT<R>::V twk(typename CT<R>::V b, int k) {
  static_assert(192 % N == 0, "register DFT size must divide 192");
  const int q = (k % N) * (192 / N);
  if (q == 0) return b;
  if (q == 48) return mk(b.y, -b.x);    // -i
  if (q == 96) return mk(-b.x, -b.y);   // -1
  if (q == 144) return mk(-b.y, b.x);   // +i
  if (q == 24 || q == 72 || q == 120 || q == 168) {
    typename CT<R>::V w = w192<R>(q);  // (+-1 +- i)/sqrt2
    const R h = w.x > 0 ? w.x : -w.x;
    const R sx = w.x > 0 ? R(1) : R(-1), sy = w.y > 0 ? R(1) : R(-1);
    // (bx + i by)(sx + i sy) h
    return mk((sx * b.x - sy * b.y) * h, (sx * b.y + sy * b.x) * h);
  }
  return cmul(b, w192<R>(q));
}

// ----------------------------------------------------------------------------
// register DFTs (forward, unnormalised), sizes N | 192, mixed radix 3/4/2
// ----------------------------------------------------------------------------
template <typename V> __device__ __forceinline__ void dft2(V* a) {
  V t = a[0];
  a[0] = cadd(t, a[1]);
  a[1] = csub(t, a[1]);
}
template <typename V> __device__ __forceinline__ void dft4(V* a) {
  V t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
  V t2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
  V t3 = mk(d.y, -d.x);  // (a1 - a3) * (-i)
  a[0] = cadd(t0, t2);
  a[1] = cadd(t1, t3);
  a[2] = csub(t0, t2);
  a[3] = csub(t1, t3);
}
template <typename V> __device__ __forceinline__ void dft3(V* a) {
  using R = decltype(a[0].x);
  const R c = R(0.86602540378443864676372317075293618);  // sin(2pi/3)
  V t1 = cadd(a[1], a[2]);
  V d = csub(a[1], a[2]);
  V t2 = mk(a[0].x - R(0.5) * t1.x, a[0].y - R(0.5) * t1.y);
  V t3 = mk(c * d.y, -c * d.x);  // -i * sin(2pi/3) * (a1 - a2)
  a[0] = cadd(a[0], t1);
  a[1] = cadd(t2, t3);
  a[2] = csub(t2, t3);
}

template <int N> struct RegPlan {
  static constexpr int has3 = (N % 3 == 0) ? 1 : 0;
  static constexpr int P = has3 ? N / 3 : N;
  static constexpr int lg = (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : (P >= 2) ? 1 : 0;
  static constexpr int n4 = lg / 2, n2 = lg % 2;
  static constexpr int NST = has3 + n4 + n2;
  static constexpr int radix(int i) { return (has3 && i == 0) ? 3 : (i < has3 + n4) ? 4 : 2; }
};

template <typename R, int N, int I, int NS>
__device__ __forceinline__ void reg_stage(typename CT<R>::V* v) {
  using V = typename CT<R>::V;
  if constexpr (I < RegPlan<N>::NST) {
    constexpr int r = RegPlan<N>::radix(I);
    V o[N];
#pragma unroll
    for (int j = 0; j < N / r; ++j) {
      const int k = j % NS;
      V a[r];
#pragma unroll
      for (int t = 0; t < r; ++t) a[t] = twk<R, NS * r>(v[j + t * (N / r)], k * t);
      if constexpr (r == 2) dft2(a);
      if constexpr (r == 3) dft3(a);
      if constexpr (r == 4) dft4(a);
#pragma unroll
      for (int t = 0; t < r; ++t) o[(j - k) * r + k + t * NS] = a[t];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = o[j];
    reg_stage<R, N, I + 1, NS * r>(v);
  }
}

template <typename R, int N>
__device__ __forceinline__ void reg_dft(typename CT<R>::V* v) {
  if constexpr (N > 1) reg_stage<R, N, 0, 1>(v);
}

// ----------------------------------------------------------------------------
// pass descriptors (host-built, passed by value)
// ----------------------------------------------------------------------------
struct SubDesc {
  int64_t ncols, cg, cs;        // column validity: grp*cg + s*cs + f < ncols
  int64_t ig, it, if_, is, im;  // load offsets (elements)
  int64_t og, ot, of, os, om;   // store offsets (elements)
  int64_t tw_mod;               // modulus of the fused DIT twiddle, 0 = none
  int64_t Ag, At, Af, As;       // A = grp*Ag + task*At + f*Af + s*As
  int64_t C0, Ct, Cs, Cm;       // C = C0 + task*Ct + s*Cs + m*Cm ; e = A*C mod tw_mod
  int32_t ntasks;               // tasks per column group
  int32_t in_staging, out_staging;
  int32_t store_mode;           // 0 direct (f fastest), 1 s fastest, 2 m fastest (via smem)
  int32_t conj_in, conj_out, check_finite, pad_;
  double scale;                 // output scale (1 = none)
};

struct PassArgs {
  const void* in;
  void* out;
  void* staging;
  int64_t slot_elems;  // elements per staging slot (one column group)
  SubDesc a, b;
  int64_t ngroups;
  int64_t total_tasks;
  int32_t nslots, lag, staged, pad_;
  unsigned long long* task_counter;
  int32_t* doneA;
  int32_t* doneB;
  int32_t* flag;  // bit 0: non-finite input seen
};

// e = A*C mod M for M = 2^k or 3*2^k (A, C >= 0), exact.
__device__ __forceinline__ int64_t mulmod(int64_t A, int64_t C, int64_t M) {
  const uint64_t lo = (uint64_t)A * (uint64_t)C;  // exact mod 2^64
  if ((M & (M - 1)) == 0) return (int64_t)(lo & (uint64_t)(M - 1));
  const int k = __ffsll(M) - 1;  // M = 3 * 2^k
  const uint64_t p2 = lo & ((1ull << k) - 1);
  const int m3 = (int)(((A % 3) * (C % 3)) % 3);
  const int inv = (k & 1) ? 2 : 1;  // (2^k)^-1 mod 3
  const int y = (((m3 - (int)(p2 % 3)) % 3 + 3) * inv) % 3;
  return (int64_t)(p2 + ((uint64_t)y << k));
}

// W_M^e = exp(-2 pi i e / M) in fp64.
__device__ __forceinline__ double2 wroot(int64_t e, int64_t M) {
  double s, c;
  sincospi(-2.0 * ((double)e / (double)M), &s, &c);
  return make_double2(c, s);
}

// ----------------------------------------------------------------------------
// in-CTA stage plan: radices sigma_i | E, prod sigma_i = RHO
// ----------------------------------------------------------------------------
struct StagePlan {
  int n;
  int sig[12];
};
constexpr StagePlan make_stage_plan(int rho, int e) {
  StagePlan p{0, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
  const int cand[9] = {32, 24, 16, 12, 8, 6, 4, 3, 2};
  int rem = rho;
  while (rem > 1) {
    int pick = 0;
    for (int i = 0; i < 9; ++i)
      if (rem % cand[i] == 0 && e % cand[i] == 0) {
        pick = cand[i];
        break;
      }
    if (pick == 0) return StagePlan{-1, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
    p.sig[p.n++] = pick;
    rem /= pick;
  }
  if (p.n == 0) p.sig[p.n++] = 1;
  return p;
}

template <typename R, int RHO_, int D_, int NT_>
struct Tile {
  using V = typename CT<R>::V;
  static constexpr int RHO = RHO_, D = D_, NT = NT_;
  static constexpr int F = CT<R>::F;
  static constexpr int TILE = F * D * RHO;
  static constexpr int E = TILE / NT;
  static_assert(E * NT == TILE, "tile must split evenly over threads");
  static constexpr StagePlan PL = make_stage_plan(RHO, E);
  static_assert(PL.n > 0, "no stage plan for this tile");
  static constexpr int NST = PL.n;
  static constexpr int SMEM_ELEMS = D * RHO * (F + 1);

  __device__ __forceinline__ static int sidx(int f, int s, int m) { return (m * D + s) * (F + 1) + f; }

  static constexpr int prod_before(int i) {
    int p = 1;
    for (int k = 0; k < i; ++k) p *= PL.sig[k];
    return p;
  }

  // per-CTA table W_RHO^i, i < RHO, fp64 sincospi then rounded once
  __device__ static void build_table(V* tw) {
    for (int i = threadIdx.x; i < RHO; i += blockDim.x) tw[i] = to_v(wroot(i, RHO), R());
  }

  template <int I>
  __device__ __forceinline__ static void stage_compute(V* v, const V* tw) {
    constexpr int S = PL.sig[I];
    constexpr int Q = E / S;
    constexpr int L = RHO / S;
    constexpr int NS = prod_before(I);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if constexpr (I > 0 && NS > 1) {
        const int g = threadIdx.x + q * NT;
        const int u = (g / F) % L;
        const int k = u % NS;
        constexpr int STEP = RHO / (NS * S);
#pragma unroll
        for (int t = 1; t < S; ++t) v[q * S + t] = cmul(v[q * S + t], tw[k * t * STEP]);
      }
      reg_dft<R, S>(v + q * S);
    }
  }

  template <int I>
  __device__ __forceinline__ static void stage_write(V* v, V* sm) {
    constexpr int S = PL.sig[I];
    constexpr int Q = E / S;
    constexpr int L = RHO / S;
    constexpr int NS = prod_before(I);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int g = threadIdx.x + q * NT;
      const int f = g % F, x = g / F, u = x % L, s = x / L;
      const int k = u % NS;
#pragma unroll
      for (int t = 0; t < S; ++t) sm[sidx(f, s, (u - k) * S + k + t * NS)] = v[q * S + t];
    }
  }

  template <int I>
  __device__ __forceinline__ static void stage_read(V* v, const V* sm) {
    constexpr int S = PL.sig[I];
    constexpr int Q = E / S;
    constexpr int L = RHO / S;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int g = threadIdx.x + q * NT;
      const int f = g % F, x = g / F, u = x % L, s = x / L;
#pragma unroll
      for (int t = 0; t < S; ++t) v[q * S + t] = sm[sidx(f, s, u + t * L)];
    }
  }

  template <int I>
  __device__ __forceinline__ static void stages(V* v, V* sm, const V* tw) {
    if constexpr (I < NST) {
      if constexpr (I > 0) {
        stage_read<I>(v, sm);
        __syncthreads();
      }
      stage_compute<I>(v, tw);
      if constexpr (I + 1 < NST) {
        stage_write<I>(v, sm);
        __syncthreads();
      }
      stages<I + 1>(v, sm, tw);
    }
  }

  // One tile: load (+conj, +finite check, +DIT twiddle), RHO-point DFTs, store.
  __device__ static void run(const SubDesc& d, const PassArgs& p, int64_t grp, int task, V* sm,
                             const V* tw, bool& nonfinite) {
    V v[E];
    constexpr int S0 = PL.sig[0];
    constexpr int Q0 = E / S0;
    constexpr int L0 = RHO / S0;
    const V* src = d.in_staging
                       ? (const V*)p.staging + (grp % p.nslots) * p.slot_elems + task * d.it
                       : (const V*)p.in + grp * d.ig + task * d.it;
    // ---- load in the stage-0 arrangement (f fastest: 128-byte runs)
#pragma unroll
    for (int q = 0; q < Q0; ++q) {
      const int g = threadIdx.x + q * NT;
      const int f = g % F, x = g / F, u = x % L0, s = x / L0;
      const bool valid = grp * d.cg + s * d.cs + f < d.ncols;
      const V* bp = src + f * d.if_ + s * d.is + u * d.im;
#pragma unroll
      for (int t = 0; t < S0; ++t) {
        V x0 = mk(R(0), R(0));
        if (valid) x0 = d.in_staging ? __ldcg(bp + (int64_t)t * L0 * d.im) : __ldg(bp + (int64_t)t * L0 * d.im);
        if (d.conj_in) x0.y = -x0.y;
        if (d.check_finite && !(isfinite(x0.x) && isfinite(x0.y))) nonfinite = true;
        v[q * S0 + t] = x0;
      }
      if (d.tw_mod) {
        const int64_t M = d.tw_mod;
        const int64_t A = grp * d.Ag + task * d.At + f * d.Af + s * d.As;
        const int64_t C = d.C0 + task * d.Ct + s * d.Cs + (int64_t)u * d.Cm;
        double2 w = wroot(mulmod(A, C, M), M);
        const double2 st = wroot(mulmod(A, d.Cm * L0, M), M);
#pragma unroll
        for (int t = 0; t < S0; ++t) {
          v[q * S0 + t] = cmul(v[q * S0 + t], to_v(w, R()));
          if (t + 1 < S0) w = cmul(w, st);
        }
      }
    }
    // ---- in-CTA radix stages
    stages<0>(v, sm, tw);
    // ---- store (last stage holds m' = u + t*L for its butterflies)
    constexpr int SL = PL.sig[NST - 1];
    constexpr int QL = E / SL;
    constexpr int LL = RHO / SL;
    V* dst = d.out_staging ? (V*)p.staging + (grp % p.nslots) * p.slot_elems + task * d.ot
                           : (V*)p.out + grp * d.og + task * d.ot;
    const R sc = (R)d.scale;
    if (d.store_mode == 0) {
#pragma unroll
      for (int q = 0; q < QL; ++q) {
        const int g = threadIdx.x + q * NT;
        const int f = g % F, x = g / F, u = x % LL, s = x / LL;
        if (grp * d.cg + s * d.cs + f >= d.ncols) continue;
        V* bp = dst + f * d.of + s * d.os + u * d.om;
#pragma unroll
        for (int t = 0; t < SL; ++t) {
          V y = v[q * SL + t];
          if (d.conj_out) y.y = -y.y;
          if (d.scale != 1.0) y = mk(y.x * sc, y.y * sc);
          if (d.out_staging)
            __stcg(bp + (int64_t)t * LL * d.om, y);
          else
            bp[(int64_t)t * LL * d.om] = y;
        }
      }
    } else {
      // transpose through shared memory so the output's unit-stride index is fastest
#pragma unroll
      for (int q = 0; q < QL; ++q) {
        const int g = threadIdx.x + q * NT;
        const int f = g % F, x = g / F, u = x % LL, s = x / LL;
#pragma unroll
        for (int t = 0; t < SL; ++t) sm[sidx(f, s, u + t * LL)] = v[q * SL + t];
      }
      __syncthreads();
#pragma unroll 4
      for (int q = 0; q < E; ++q) {
        const int o = threadIdx.x + q * NT;
        int f, s, m;
        if (d.store_mode == 1) {
          s = o % D;
          f = (o / D) % F;
          m = o / (D * F);
        } else {
          m = o % RHO;
          s = (o / RHO) % D;
          f = o / (RHO * D);
        }
        if (grp * d.cg + s * d.cs + f >= d.ncols) continue;
        V y = sm[sidx(f, s, m)];
        if (d.conj_out) y.y = -y.y;
        if (d.scale != 1.0) y = mk(y.x * sc, y.y * sc);
        V* ptr = dst + f * d.of + s * d.os + (int64_t)m * d.om;
        if (d.out_staging)
          __stcg(ptr, y);
        else
          *ptr = y;
      }
    }
  }
};

// Empty B-tile marker for direct (un-staged) passes.
struct NoTile {
  static constexpr int SMEM_ELEMS = 0, RHO = 0, NT = 0;
};

__device__ __forceinline__ void wait_at_least(const int32_t* ctr, int32_t need) {
  if (threadIdx.x == 0) {
    while (*(volatile const int32_t*)ctr < need) __nanosleep(128);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void signal_done(int32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
  }
}

// Persistent pass kernel: CTAs pull tasks from one global counter in a fixed
// order (A(0..lag-1), then B(g-lag), A(g) pairs, then the tail of B), which
// makes every wait target a task that an already-running CTA owns.
template <typename R, class TA, class TB>
__global__ void __launch_bounds__(TA::NT) pass_kernel(const PassArgs p) {
  using V = typename CT<R>::V;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int SM_ELEMS = TA::SMEM_ELEMS > TB::SMEM_ELEMS ? TA::SMEM_ELEMS : TB::SMEM_ELEMS;
  V* sm = reinterpret_cast<V*>(smem_raw);
  V* twA = sm + SM_ELEMS;
  V* twB = twA + TA::RHO;
  __shared__ unsigned long long s_task;
  TA::build_table(twA);
  if constexpr (TB::RHO > 0) TB::build_table(twB);
  bool nonfinite = false;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(p.task_counter, 1ull);
    __syncthreads();
    const int64_t pos = (int64_t)s_task;
    if (pos >= p.total_tasks) break;
    if (!p.staged) {
      const int64_t grp = pos / p.a.ntasks;
      TA::run(p.a, p, grp, (int)(pos % p.a.ntasks), sm, twA, nonfinite);
      __syncthreads();
      continue;
    }
    if constexpr (TB::RHO > 0) {
      const int64_t G = p.ngroups, L = p.lag, TAn = p.a.ntasks, TBn = p.b.ntasks;
      bool isB;
      int64_t grp, sub;
      if (pos < L * TAn) {
        isB = false;
        grp = pos / TAn;
        sub = pos % TAn;
      } else if (pos < L * TAn + (G - L) * (TAn + TBn)) {
        const int64_t q = pos - L * TAn;
        const int64_t i = L + q / (TAn + TBn), r = q % (TAn + TBn);
        if (r < TBn) {
          isB = true;
          grp = i - L;
          sub = r;
        } else {
          isB = false;
          grp = i;
          sub = r - TBn;
        }
      } else {
        const int64_t q = pos - L * TAn - (G - L) * (TAn + TBn);
        isB = true;
        grp = G - L + q / TBn;
        sub = q % TBn;
      }
      if (!isB) {
        if (grp >= p.nslots) wait_at_least(p.doneB + (grp - p.nslots), (int32_t)TBn);
        TA::run(p.a, p, grp, (int)sub, sm, twA, nonfinite);
        signal_done(p.doneA + grp);
      } else {
        wait_at_least(p.doneA + grp, (int32_t)TAn);
        TB::run(p.b, p, grp, (int)sub, sm, twB, nonfinite);
        signal_done(p.doneB + grp);
      }
    }
  }
  if (__syncthreads_or(nonfinite) && threadIdx.x == 0) atomicOr(p.flag, 1);
}

}  // namespace efft

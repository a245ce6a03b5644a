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
// sizeof(complex) = 128 B: every global access is a full 128-byte line read as
// eight 16-byte vectors), D independent DFTs, RHO points each.  The tile lives
// in registers (E elements per thread) and is exchanged through shared memory
// rows padded to 144 B (16-byte aligned, conflict-free for row-, column- and
// transposed accesses) between the in-CTA radix stages.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <type_traits>

#include "w192_table.cuh"
#include "w320_table.cuh"
#include "w448_table.cuh"

namespace efft {

// ----------------------------------------------------------------------------
// compile-time loop
// ----------------------------------------------------------------------------
template <int I, int E, class Fn>
__device__ __forceinline__ void cfor(Fn&& f) {
  if constexpr (I < E) {
    f(std::integral_constant<int, I>{});
    cfor<I + 1, E>(f);
  }
}

// ----------------------------------------------------------------------------
// complex helpers
// ----------------------------------------------------------------------------
template <typename R> struct CT;
template <> struct CT<float> {
  using V = float2;                 // one complex element
  static constexpr int F = 16;      // columns per 128-byte row
  static constexpr int VEC = 2;     // default elements per lane access (16 bytes)
};
template <> struct CT<double> {
  using V = double2;
  static constexpr int F = 8;
  static constexpr int VEC = 1;
};

// access vector of VEC adjacent complex elements (one lane's global/smem access)
template <typename R, int VEC> struct VecT;
template <> struct VecT<float, 2> { using T = float4; };
template <> struct VecT<float, 1> { using T = float2; };
template <> struct VecT<double, 1> { using T = double2; };

__device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }

// ---- paired-fp32 (sm_100 FADD2 / FMUL2 / FFMA2) complex64 arithmetic: one
// instruction per complex add, two per complex multiply; ptxas folds the
// broadcast (x, x) / swapped (y, x) operand pairs into operand selectors.
typedef unsigned long long u64;
__device__ __forceinline__ u64 p64(float2 a) {
  u64 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a.x), "f"(a.y));
  return d;
}
__device__ __forceinline__ float2 f64p(u64 a) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(a));
  return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p64(a)), "l"(p64(b)));
  return f64p(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p64(a)), "l"(p64(b)));
  return f64p(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p64(a)), "l"(p64(b)));
  return f64p(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {  // a*b + c per lane
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(p64(a)), "l"(p64(b)), "l"(p64(c)));
  return f64p(d);
}

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return mk(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return mk(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <> __device__ __forceinline__ float2 cadd<float2>(float2 a, float2 b) { return add2(a, b); }
template <> __device__ __forceinline__ float2 csub<float2>(float2 a, float2 b) { return sub2(a, b); }
template <> __device__ __forceinline__ float2 cmul<float2>(float2 a, float2 b) {
  // (a.x b.x - a.y b.y, a.x b.y + a.y b.x) = (a.x,a.x)*(b.x,b.y) + (a.y,a.y)*(-b.y,b.x)
  return fma2(make_float2(a.y, a.y), make_float2(-b.y, b.x), mul2(make_float2(a.x, a.x), b));
}
// a + (-i) d and a - (-i) d (the radix-4 rotation fused into the add)
__device__ __forceinline__ double2 add_mi(double2 a, double2 d) { return mk(a.x + d.y, a.y - d.x); }
__device__ __forceinline__ double2 sub_mi(double2 a, double2 d) { return mk(a.x - d.y, a.y + d.x); }
__device__ __forceinline__ float2 add_mi(float2 a, float2 d) {
  return fma2(make_float2(d.y, d.x), make_float2(1.f, -1.f), a);
}
__device__ __forceinline__ float2 sub_mi(float2 a, float2 d) {
  return fma2(make_float2(d.y, d.x), make_float2(-1.f, 1.f), a);
}
__device__ __forceinline__ float2 to_v(double2 w, float) { return make_float2((float)w.x, (float)w.y); }
__device__ __forceinline__ double2 to_v(double2 w, double) { return w; }

// 16-byte vector <-> VEC complex elements
__device__ __forceinline__ void unpack(float4 a, float2* v0, float2* v1) {
  *v0 = make_float2(a.x, a.y);
  *v1 = make_float2(a.z, a.w);
}
__device__ __forceinline__ float4 pack(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }

// ----------------------------------------------------------------------------
// 16-byte global accesses with L2 eviction-priority hints.  The array being
// transformed streams through L2 once per pass (evict_first); the staging ring
// must stay resident between its producer and consumer tiles (evict_last), and
// is discarded (no write-back) once consumed.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <typename VT>
__device__ __forceinline__ VT ld_stream(const VT* ptr, uint64_t pol) {
  if constexpr (sizeof(VT) == 16) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr), "l"(pol));
    return *reinterpret_cast<VT*>(&r);
  } else {
    static_assert(sizeof(VT) == 8, "8- or 16-byte accesses");
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(ptr), "l"(pol));
    return *reinterpret_cast<VT*>(&r);
  }
}
template <typename VT>
__device__ __forceinline__ VT ld_staging(const VT* ptr) {
  if constexpr (sizeof(VT) == 16) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr));
    return *reinterpret_cast<VT*>(&r);
  } else {
    uint2 r;
    asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(ptr));
    return *reinterpret_cast<VT*>(&r);
  }
}
template <typename VT>
__device__ __forceinline__ void st_hint(VT* ptr, VT v, uint64_t pol) {
  if constexpr (sizeof(VT) == 16) {
    const uint4 u = *reinterpret_cast<const uint4*>(&v);
    asm volatile("st.global.cg.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(ptr), "r"(u.x), "r"(u.y),
                 "r"(u.z), "r"(u.w), "l"(pol)
                 : "memory");
  } else {
    static_assert(sizeof(VT) == 8, "8- or 16-byte accesses");
    const uint2 u = *reinterpret_cast<const uint2*>(&v);
    asm volatile("st.global.cg.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;" ::"l"(ptr), "r"(u.x), "r"(u.y), "l"(pol)
                 : "memory");
  }
}
// Drop a consumed 128-byte staging line from L2 without writing it back.
__device__ __forceinline__ void l2_discard(const void* ptr) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(ptr) : "memory");
}

// ----------------------------------------------------------------------------
// mbarrier + bulk asynchronous copy (TMA engine, cp.async.bulk) primitives
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking poll (test_wait never suspends the thread)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait with a watchdog: after ~2^28 polls report who is stuck and trap
__device__ __forceinline__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int tag, long long a, long long b) {
  long long n = 0;
  while (!mbar_try(bar, parity)) {
    if (++n == (1ll << 30)) {
      printf("EFFT STUCK tag=%d cta=%d thr=%d parity=%u a=%lld b=%lld\n", tag, blockIdx.x, threadIdx.x, parity, a, b);
      __trap();
    }
  }
}
// global -> shared bulk copy completing `bytes` transactions on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// TMA tensor copies (one instruction per box), 128B-swizzled into shared memory
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void red_release_add(int32_t* ctr, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(ctr), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire(const int32_t* ctr) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  return v;
}
// order generic-proxy writes observed through an acquire before async-proxy reads
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// b * W_N^K for N | T (T = 320 or 448, table W): trivial roots become sign
// swaps, the rest immediate-operand complex multiplies.
template <typename R, int N, int K, int T, class W>
__device__ __forceinline__ typename CT<R>::V twk_tab(typename CT<R>::V b) {
  static_assert(T % N == 0, "register DFT size must divide the root table");
  constexpr int Q = (K % N) * (T / N);
  if constexpr (Q == 0) {
    return b;
  } else if constexpr (4 * Q == T) {
    return mk(b.y, -b.x);  // -i
  } else if constexpr (2 * Q == T) {
    return mk(-b.x, -b.y);
  } else if constexpr (4 * Q == 3 * T) {
    return mk(-b.y, b.x);  // +i
  } else {
    constexpr R wr = (R)W::v[Q][0], wi = (R)W::v[Q][1];
    if constexpr (sizeof(R) == 4)
      return fma2(make_float2(b.y, b.y), make_float2(-wi, wr), mul2(make_float2(b.x, b.x), make_float2(wr, wi)));
    else
      return mk(fma(b.x, wr, -b.y * wi), fma(b.x, wi, b.y * wr));
  }
}
// b * W_N^K, N | 192, 320 or 448, K compile-time
template <typename R, int N, int K>
__device__ __forceinline__ typename CT<R>::V twk(typename CT<R>::V b) {
  if constexpr (192 % N != 0) {
    if constexpr (320 % N == 0)
      return twk_tab<R, N, K, 320, W320>(b);
    else
      return twk_tab<R, N, K, 448, W448>(b);
  } else {
  static_assert(192 % N == 0, "register DFT size must divide 192");
  constexpr int Q = (K % N) * (192 / N);
  if constexpr (Q == 0) {
    return b;
  } else if constexpr (Q == 48) {
    return mk(b.y, -b.x);  // -i
  } else if constexpr (Q == 96) {
    return mk(-b.x, -b.y);
  } else if constexpr (Q == 144) {
    return mk(-b.y, b.x);  // +i
  } else if constexpr (Q == 24 || Q == 72 || Q == 120 || Q == 168) {
    constexpr R h = (R)0.70710678118654752440084436210484903928;
    if constexpr (sizeof(R) == 4) {
      // h*(b + (-i)b) etc: one FFMA2 for the rotation-add, one FMUL2 for the scale
      if constexpr (Q == 24) return mul2(add_mi(b, b), make_float2(h, h));   // (1 - i)/sqrt2
      if constexpr (Q == 72) return mul2(sub_mi(b, b), make_float2(-h, -h));  // (-1 - i)/sqrt2
      if constexpr (Q == 120) return mul2(add_mi(b, b), make_float2(-h, -h));  // (-1 + i)/sqrt2 = -(1 - i)/sqrt2
      if constexpr (Q == 168) return mul2(sub_mi(b, b), make_float2(h, h));   // (1 + i)/sqrt2
    } else {
      if constexpr (Q == 24) return mk((b.x + b.y) * h, (b.y - b.x) * h);
      if constexpr (Q == 72) return mk((b.y - b.x) * h, -(b.x + b.y) * h);
      if constexpr (Q == 120) return mk(-(b.x + b.y) * h, (b.x - b.y) * h);
      if constexpr (Q == 168) return mk((b.x - b.y) * h, (b.x + b.y) * h);
    }
  } else {
    constexpr R wr = (R)W192::v[Q][0], wi = (R)W192::v[Q][1];
    if constexpr (sizeof(R) == 4)
      return fma2(make_float2(b.y, b.y), make_float2(-wi, wr), mul2(make_float2(b.x, b.x), make_float2(wr, wi)));
    else
      return mk(fma(b.x, wr, -b.y * wi), fma(b.x, wi, b.y * wr));
  }
  }
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
  a[0] = cadd(t0, t2);
  a[1] = add_mi(t1, d);  // t1 + (a1 - a3)(-i)
  a[2] = csub(t0, t2);
  a[3] = sub_mi(t1, d);
}
template <typename V> __device__ __forceinline__ void dft3(V* a) {
  using R = decltype(a[0].x);
  constexpr R c = R(0.86602540378443864676372317075293618);  // sin(2pi/3)
  V t1 = cadd(a[1], a[2]);
  V d = csub(a[1], a[2]);
  V t2 = mk(a[0].x - R(0.5) * t1.x, a[0].y - R(0.5) * t1.y);
  V t3 = mk(c * d.y, -c * d.x);  // -i * sin(2pi/3) * (a1 - a2)
  a[0] = cadd(a[0], t1);
  a[1] = cadd(t2, t3);
  a[2] = csub(t2, t3);
}

// 5-point DFT (forward): pairs (1,4), (2,3) with c_k = cos(2 pi k/5),
// s_k = sin(2 pi k/5); X_1,4 = a0 + c1 t1 + c2 t2 -/+ i (s1 d1 + s2 d2),
// X_2,3 = a0 + c2 t1 + c1 t2 -/+ i (s2 d1 - s1 d2).
template <typename V> __device__ __forceinline__ void dft5(V* a) {
  using R = decltype(a[0].x);
  constexpr R c1 = R(0.30901699437494742410229341718281905886);
  constexpr R c2 = R(-0.80901699437494742410229341718281905886);
  constexpr R s1 = R(0.95105651629515357211643933337938214340);
  constexpr R s2 = R(0.58778525229247312916870595463907276860);
  const V t1 = cadd(a[1], a[4]), d1 = csub(a[1], a[4]);
  const V t2 = cadd(a[2], a[3]), d2 = csub(a[2], a[3]);
  const V a0 = a[0];
  const V u1 = mk(a0.x + c1 * t1.x + c2 * t2.x, a0.y + c1 * t1.y + c2 * t2.y);
  const V u2 = mk(a0.x + c2 * t1.x + c1 * t2.x, a0.y + c2 * t1.y + c1 * t2.y);
  const V w1 = mk(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
  const V w2 = mk(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
  a[0] = cadd(a0, cadd(t1, t2));
  a[1] = mk(u1.x + w1.y, u1.y - w1.x);  // u1 - i w1
  a[4] = mk(u1.x - w1.y, u1.y + w1.x);  // u1 + i w1
  a[2] = mk(u2.x + w2.y, u2.y - w2.x);
  a[3] = mk(u2.x - w2.y, u2.y + w2.x);
}

// 7-point DFT (forward): X_k = a0 + sum_{j=1..3} [c_jk (a_j + a_7-j) - i s_jk (a_j - a_7-j)]
// with c_m = cos(2 pi m/7), s_m = sin(2 pi m/7) (compile-time, from W_448).
template <typename V> __device__ __forceinline__ void dft7(V* a) {
  using R = decltype(a[0].x);
  V t[4], d[4];
  cfor<1, 4>([&](auto J) {
    constexpr int j = decltype(J)::value;
    t[j] = cadd(a[j], a[7 - j]);
    d[j] = csub(a[j], a[7 - j]);
  });
  const V a0 = a[0];
  a[0] = cadd(a0, cadd(t[1], cadd(t[2], t[3])));
  cfor<1, 4>([&](auto K) {
    constexpr int k = decltype(K)::value;
    V u = a0, w = mk(R(0), R(0));
    cfor<1, 4>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int m = (j * k) % 7;
      constexpr R c = (R)W448::v[64 * m][0], sn = (R)(-W448::v[64 * m][1]);
      u = mk(u.x + c * t[j].x, u.y + c * t[j].y);
      w = mk(w.x + sn * d[j].x, w.y + sn * d[j].y);
    });
    a[k] = mk(u.x + w.y, u.y - w.x);      // u - i w
    a[7 - k] = mk(u.x - w.y, u.y + w.x);  // u + i w
  });
}

// In-place decimation-in-frequency network over a contiguous segment
// [B, B+L) of v: radix r = 3 (if 3 | L), else 5, else 7, else 4, else 2; twiddles
// W_L^(j*k) are compile-time constants.  Output X[k] ends at v[dif_pos<N>(k)]
// (mixed-radix digit reversal; free renaming, no register copies).
constexpr int dif_radix_rt(int L) {
  return (L % 3 == 0) ? 3 : (L % 5 == 0) ? 5 : (L % 7 == 0) ? 7 : (L % 4 == 0) ? 4 : 2;
}
constexpr int dif_pos(int L, int k) {
  // position of output k of an L-point in-place DIF transform
  int pos = 0;
  while (L > 1) {
    const int r = dif_radix_rt(L);
    const int q = L / r;
    pos += (k % r) * q;
    k /= r;
    L = q;
  }
  return pos;
}
// Same map with L a template parameter: every radix and stride is a
// compile-time constant, so with k from an unrolled loop the position folds
// to an immediate (register arrays stay in registers whatever the radix set).
template <int L>
__device__ __forceinline__ constexpr int dif_pos_t(int k) {
  if constexpr (L <= 1) {
    return 0;
  } else {
    constexpr int r = dif_radix_rt(L), q = L / r;
    return (k % r) * q + dif_pos_t<q>(k / r);
  }
}

template <typename R, int L, int B>
__device__ __forceinline__ void dif_segment(typename CT<R>::V* v) {
  using V = typename CT<R>::V;
  if constexpr (L > 1) {
    constexpr int r = dif_radix_rt(L);
    constexpr int q = L / r;
    cfor<0, q>([&](auto J) {
      constexpr int j = decltype(J)::value;
      V a[r];
      cfor<0, r>([&](auto T) { a[decltype(T)::value] = v[B + j + decltype(T)::value * q]; });
      if constexpr (r == 2) dft2(a);
      if constexpr (r == 3) dft3(a);
      if constexpr (r == 4) dft4(a);
      if constexpr (r == 5) dft5(a);
      if constexpr (r == 7) dft7(a);
      cfor<0, r>([&](auto T) {
        constexpr int k = decltype(T)::value;
        v[B + j + k * q] = twk<R, L, j * k>(a[k]);
      });
    });
    cfor<0, r>([&](auto T) { dif_segment<R, q, B + decltype(T)::value * q>(v); });
  }
}

template <typename R, int N>
__device__ __forceinline__ void reg_dft(typename CT<R>::V* v) {
  dif_segment<R, N, 0>(v);
}

// ----------------------------------------------------------------------------
// pass descriptors (host-built, passed by value as a __grid_constant__)
// ----------------------------------------------------------------------------
struct SubDesc {
  int64_t ncols, cg, cs;   // column validity: grp*cg + s*cs + f < ncols
  int64_t ig, it, is, im;  // load offsets (elements); columns are unit stride
  int64_t og, ot, of, os, om;  // store offsets (elements)
  int64_t tw_mod;          // modulus of the fused DIT twiddle, 0 = none
  int64_t A0, Ag, At, Af, As;  // A = A0 + grp*Ag + task*At + f*Af + s*As
  int64_t C0, Ct, Cs, Cm;  // C = C0 + task*Ct + s*Cs + m*Cm ; e = A*C mod tw_mod
  int32_t ntasks;          // tasks per column group
  int32_t in_staging, out_staging;
  int32_t store_mode;      // 0 direct (f unit stride), 1 s unit stride, 2 m unit stride
  int32_t conj_in, conj_out, check_finite, pad_;
  double scale;            // output scale (applied with conj_out)
};

struct PassArgs {
  const void* in;
  void* out;
  void* staging;
  int64_t slot_elems;  // elements per staging slot (one column group)
  SubDesc a, b;
  int64_t ngroups;
  int64_t total_tasks;
  int32_t nslots, lag, staged, nowait;  // nowait: diagnostic only (skips dependency waits)
  unsigned long long* task_counter;
  int32_t* doneA;
  int32_t* doneB;
  int32_t* flag;  // bit 0: non-finite input seen
  // TMA maps of the warp-specialised staged kernel: A tiles read the pass
  // input [column, u, t]; B tiles read the staging ring [f, k1, u, slot]
  alignas(64) CUtensorMap tmA;
  alignas(64) CUtensorMap tmB;
};

// e = A*C mod M for M = m*2^k, m in {1, 3, 5, 7} (A, C >= 0), exact: the low k
// bits come from the 64-bit product, the residue mod m by CRT.
__device__ __forceinline__ int64_t mulmod(int64_t A, int64_t C, int64_t M) {
  const uint64_t lo = (uint64_t)A * (uint64_t)C;  // exact mod 2^64
  if ((M & (M - 1)) == 0) return (int64_t)(lo & (uint64_t)(M - 1));
  const int k = __ffsll(M) - 1;  // M = m * 2^k
  const int m = (int)(M >> k);
  const uint64_t p2 = lo & ((1ull << k) - 1);
  const int mm = (int)(((A % m) * (C % m)) % m);
  int pw = 1;  // 2^k mod m, then its inverse
  for (int i = 0; i < k; ++i) pw = (2 * pw) % m;
  int inv = 1;
  while ((inv * pw) % m != 1) ++inv;
  const int y = (((mm - (int)(p2 % m)) % m + m) * inv) % m;
  return (int64_t)(p2 + ((uint64_t)y << k));
}

// W_M^e = exp(-2 pi i e / M) in fp64.
__device__ __forceinline__ double2 wroot(int64_t e, int64_t M) {
  double s, c;
  sincospi(-2.0 * ((double)e / (double)M), &s, &c);
  return make_double2(c, s);
}

// ----------------------------------------------------------------------------
// in-CTA stage plan: radices sigma_i | EV, prod sigma_i = RHO
// ----------------------------------------------------------------------------
struct StagePlan {
  int n;
  int sig[12];
};
constexpr StagePlan make_stage_plan(int rho, int e) {
  StagePlan p{0, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
  const int cand[15] = {32, 28, 24, 20, 16, 14, 12, 10, 8, 7, 6, 5, 4, 3, 2};
  int rem = rho;
  while (rem > 1) {
    int pick = 0;
    for (int i = 0; i < 15; ++i)
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

template <typename R, int RHO_, int D_, int NT_, bool MASK_, int VEC_, int TOFF_ = 0, int BAR_ = 0, bool SWZ_ = false>
struct Tile {
  static constexpr int TOFF = TOFF_, BAR = BAR_;
  static constexpr bool SWZ = SWZ_;  // stage-0 input lands as dense 128B-swizzled rows (TMA)
  // tile-thread index and the barrier over the tile's threads (named barrier
  // when the tile threads are the consumer warps of a warp-specialised CTA)
  __device__ __forceinline__ static int tx() { return (int)threadIdx.x - TOFF; }
  __device__ __forceinline__ static void tsync() {
    if constexpr (BAR == 0)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT_) : "memory");
  }
  using V = typename CT<R>::V;
  static constexpr int VEC = VEC_;
  using VT = typename VecT<R, VEC>::T;
  static constexpr int RHO = RHO_, D = D_, NT = NT_;
  static constexpr bool MASK = MASK_;
  static constexpr int F = CT<R>::F;
  static constexpr int FV = F / VEC;     // lanes per 128-byte row (8)
  static constexpr int EPC = 16 / (int)sizeof(V);       // elements per 16-byte chunk
  static constexpr int PADF = F + EPC;                   // exchange row pitch: 144 bytes
  static constexpr int TILE = F * D * RHO;
  static constexpr int E = TILE / NT;    // complex elements per thread
  static constexpr int EV = E / VEC;     // butterfly elements per column-lane
  static_assert(E * NT == TILE && EV * VEC == E, "tile must split evenly over threads");
  static_assert(NT % FV == 0, "threads must cover whole rows");
  static constexpr StagePlan PL = make_stage_plan(RHO, EV);
  static_assert(PL.n > 0, "no stage plan for this tile");
  static constexpr int NST = PL.n;
  static constexpr int SMEM_ELEMS = D * RHO * PADF;

  // exchange layout: padded rows (index = base + t * const along m)
  __device__ __forceinline__ static int sidx(int f, int s, int m) { return (m * D + s) * PADF + f; }
  // TMA landing layout: dense 128-byte rows, 16-byte chunks XOR-swizzled by row % 8
  __device__ __forceinline__ static int sidx_in(int f, int s, int m) {
    const int row = m * D + s;
    return row * F + (((f / EPC) ^ (row & 7)) * EPC) + (f % EPC);
  }

  // register position of output t of an S-point in-place DFT

  static constexpr int prod_before(int i) {
    int p = 1;
    for (int k = 0; k < i; ++k) p *= PL.sig[k];
    return p;
  }

  // per-CTA table W_RHO^i, i < RHO, fp64 sincospi rounded once
  __device__ static void build_table(V* tw) {
    for (int i = threadIdx.x; i < RHO; i += blockDim.x) tw[i] = to_v(wroot(i, RHO), R());  // all CTA threads
  }

  // thread-butterfly q of a stage with radix S: (column lane, u, s)
  template <int S>
  __device__ __forceinline__ static void coords(int q, int& fv, int& u, int& s) {
    constexpr int L = RHO / S;
    const int g = tx() + q * NT;
    fv = g % FV;
    const int x = g / FV;
    u = x % L;
    s = x / L;
  }

  __device__ __forceinline__ static void put(V* sm, int f, int s, int m, const V* v0, const V* v1) {
    if constexpr (VEC == 2)
      *reinterpret_cast<VT*>(sm + sidx(f, s, m)) = pack(*v0, *v1);
    else
      sm[sidx(f, s, m)] = *v0;
  }
  __device__ __forceinline__ static void get(const V* sm, int f, int s, int m, V* v0, V* v1) {
    if constexpr (VEC == 2)
      unpack(*reinterpret_cast<const VT*>(sm + sidx(f, s, m)), v0, v1);
    else
      *v0 = sm[sidx(f, s, m)];
  }

  template <int I>
  __device__ __forceinline__ static void stage_compute(V* v, const V* tw) {
    constexpr int S = PL.sig[I];
    constexpr int Q = EV / S;
    constexpr int NS = prod_before(I);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if constexpr (I > 0) {
        int fv, u, s;
        coords<S>(q, fv, u, s);
        const int k = u % NS;
        constexpr int STEP = RHO / (NS * S);
#pragma unroll
        for (int t = 1; t < S; ++t) {
          const V w = tw[k * t * STEP];
#pragma unroll
          for (int c = 0; c < VEC; ++c) v[(q * VEC + c) * S + t] = cmul(v[(q * VEC + c) * S + t], w);
        }
      }
#pragma unroll
      for (int c = 0; c < VEC; ++c) reg_dft<R, S>(v + (q * VEC + c) * S);
    }
  }

  template <int I>
  __device__ __forceinline__ static void stage_write(const V* v, V* sm) {
    constexpr int S = PL.sig[I];
    constexpr int Q = EV / S;
    constexpr int NS = prod_before(I);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int fv, u, s;
      coords<S>(q, fv, u, s);
      const int k = u % NS;
#pragma unroll
      for (int t = 0; t < S; ++t)
        put(sm, fv * VEC, s, (u - k) * S + k + t * NS, &v[(q * VEC) * S + dif_pos_t<S>(t)],
            &v[(q * VEC + VEC - 1) * S + dif_pos_t<S>(t)]);
    }
  }

  template <int I, bool IN = false>
  __device__ __forceinline__ static void stage_read(V* v, const V* sm) {
    constexpr int S = PL.sig[I];
    constexpr int Q = EV / S;
    constexpr int L = RHO / S;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int fv, u, s;
      coords<S>(q, fv, u, s);
      if constexpr (IN) {
        // swizzle term is t-invariant when L*D % 8 == 0: base + t * L*D*F
        constexpr bool LIN = (L * D) % 8 == 0;
        const int base = sidx_in(fv * VEC, s, u);
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const int ix = LIN ? base + t * L * D * F : sidx_in(fv * VEC, s, u + t * L);
          if constexpr (VEC == 2)
            unpack(*reinterpret_cast<const VT*>(sm + ix), &v[(q * VEC) * S + t], &v[(q * VEC + 1) * S + t]);
          else
            v[(q * VEC) * S + t] = sm[ix];
        }
      } else {
#pragma unroll
        for (int t = 0; t < S; ++t)
          get(sm, fv * VEC, s, u + t * L, &v[(q * VEC) * S + t], &v[(q * VEC + VEC - 1) * S + t]);
      }
    }
  }

  template <int I>
  __device__ __forceinline__ static void stages(V* v, V* sm, const V* tw) {
    if constexpr (I < NST) {
      if constexpr (I > 0) {
        stage_read<I>(v, sm);
        tsync();
      }
      stage_compute<I>(v, tw);
      if constexpr (I + 1 < NST) {
        stage_write<I>(v, sm);
        tsync();
      }
      stages<I + 1>(v, sm, tw);
    }
  }

  // ---- stage-0 load: 16-byte vectors, columns unit stride
  template <bool CONJ, bool CHECK>
  __device__ __forceinline__ static void load(const SubDesc& d, const V* src, int64_t grp, V* v,
                                              bool& nonfinite) {
    constexpr int S0 = PL.sig[0];
    constexpr int Q0 = EV / S0;
    constexpr int L0 = RHO / S0;
    const bool stg = d.in_staging;
    const uint64_t pol = policy_evict_first();
#pragma unroll
    for (int q = 0; q < Q0; ++q) {
      int fv, u, s;
      coords<S0>(q, fv, u, s);
      const int f0 = fv * VEC;
      const V* bp = src + f0 + s * d.is + u * d.im;
      const int64_t step = (int64_t)L0 * d.im;
      bool valid[VEC];
#pragma unroll
      for (int c = 0; c < VEC; ++c) valid[c] = !MASK || grp * d.cg + s * d.cs + f0 + c < d.ncols;
#pragma unroll
      for (int t = 0; t < S0; ++t) {
        V x[VEC];
        if constexpr (MASK) {
#pragma unroll
          for (int c = 0; c < VEC; ++c) x[c] = valid[c] ? bp[c] : mk(R(0), R(0));
        } else {
          const VT* vp = reinterpret_cast<const VT*>(bp);
          const VT a = stg ? ld_staging(vp) : ld_stream(vp, pol);
          if constexpr (VEC == 2)
            unpack(a, &x[0], &x[1]);
          else
            x[0] = *reinterpret_cast<const V*>(&a);
        }
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          if constexpr (CONJ) x[c].y = -x[c].y;
          if constexpr (CHECK) nonfinite |= !(isfinite(x[c].x) && isfinite(x[c].y));
          v[(q * VEC + c) * S0 + t] = x[c];
        }
        bp += step;
      }
    }
  }

  // Every 128-byte staging row this tile read is discarded by the first lane
  // of its row (each row is consumed by exactly one tile).
  __device__ __forceinline__ static void discard_loaded(const SubDesc& d, const V* src) {
    constexpr int S0 = PL.sig[0];
    constexpr int Q0 = EV / S0;
    constexpr int L0 = RHO / S0;
#pragma unroll
    for (int q = 0; q < Q0; ++q) {
      int fv, u, s;
      coords<S0>(q, fv, u, s);
      if (fv != 0) continue;
      const V* bp = src + s * d.is + u * d.im;
      const int64_t step = (int64_t)L0 * d.im;
#pragma unroll
      for (int t = 0; t < S0; ++t) {
        l2_discard(bp);
        bp += step;
      }
    }
  }

  __device__ __forceinline__ static void twiddle(const SubDesc& d, int64_t grp, int task, V* v) {
    constexpr int S0 = PL.sig[0];
    constexpr int Q0 = EV / S0;
    constexpr int L0 = RHO / S0;
    const int64_t M = d.tw_mod;
#pragma unroll
    for (int q = 0; q < Q0; ++q) {
      int fv, u, s;
      coords<S0>(q, fv, u, s);
      const int64_t C = d.C0 + task * d.Ct + s * d.Cs + (int64_t)u * d.Cm;
      if (VEC > 1 && d.Af == 0) {  // one twiddle series serves all VEC columns
        const int64_t A = d.A0 + grp * d.Ag + task * d.At + s * d.As;
        double2 w = wroot(mulmod(A, C, M), M);
        const double2 st = wroot(mulmod(A, d.Cm * L0, M), M);
#pragma unroll
        for (int t = 0; t < S0; ++t) {
          const V wv = to_v(w, R());
#pragma unroll
          for (int c = 0; c < VEC; ++c) v[(q * VEC + c) * S0 + t] = cmul(v[(q * VEC + c) * S0 + t], wv);
          if (t + 1 < S0) w = cmul(w, st);
        }
        continue;
      }
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        const int64_t A = d.A0 + grp * d.Ag + task * d.At + (fv * VEC + c) * d.Af + s * d.As;
        double2 w = wroot(mulmod(A, C, M), M);
        const double2 st = wroot(mulmod(A, d.Cm * L0, M), M);
        V* vv = v + (q * VEC + c) * S0;
#pragma unroll
        for (int t = 0; t < S0; ++t) {
          vv[t] = cmul(vv[t], to_v(w, R()));
          if (t + 1 < S0) w = cmul(w, st);
        }
      }
    }
  }

  // ---- store, direct (f unit stride) from the last stage's registers
  template <bool CS>
  __device__ __forceinline__ static void store_direct(const SubDesc& d, V* dst, int64_t grp, const V* v) {
    constexpr int SL = PL.sig[NST - 1];
    constexpr int QL = EV / SL;
    constexpr int LL = RHO / SL;
    const R sc = (R)d.scale;
    const bool stg = d.out_staging;
    const uint64_t pol = stg ? policy_evict_last() : policy_evict_first();
#pragma unroll
    for (int q = 0; q < QL; ++q) {
      int fv, u, s;
      coords<SL>(q, fv, u, s);
      const int f0 = fv * VEC;
      V* bp = dst + f0 + s * d.os + u * d.om;
      const int64_t step = (int64_t)LL * d.om;
      bool valid[VEC];
#pragma unroll
      for (int c = 0; c < VEC; ++c) valid[c] = !MASK || grp * d.cg + s * d.cs + f0 + c < d.ncols;
#pragma unroll
      for (int t = 0; t < SL; ++t) {
        V y[VEC];
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          y[c] = v[(q * VEC + c) * SL + dif_pos_t<SL>(t)];
          if constexpr (CS) y[c] = mk(y[c].x * sc, -y[c].y * sc);
        }
        if constexpr (MASK) {
#pragma unroll
          for (int c = 0; c < VEC; ++c)
            if (valid[c]) bp[c] = y[c];
        } else if constexpr (VEC == 2) {
          st_hint(reinterpret_cast<VT*>(bp), pack(y[0], y[1]), pol);
        } else {
          st_hint(bp, y[0], pol);
        }
        bp += step;
      }
    }
  }

  // ---- store through shared memory so the output's unit-stride index is fastest
  template <bool CS, int MODE>
  __device__ __forceinline__ static void store_transposed(const SubDesc& d, V* dst, int64_t grp, const V* v,
                                                          V* sm) {
    constexpr int SL = PL.sig[NST - 1];
    constexpr int QL = EV / SL;
    constexpr int LL = RHO / SL;
#pragma unroll
    for (int q = 0; q < QL; ++q) {
      int fv, u, s;
      coords<SL>(q, fv, u, s);
#pragma unroll
      for (int t = 0; t < SL; ++t)
        put(sm, fv * VEC, s, u + t * LL, &v[(q * VEC) * SL + dif_pos_t<SL>(t)],
            &v[(q * VEC + VEC - 1) * SL + dif_pos_t<SL>(t)]);
    }
    tsync();
    constexpr int FAST = MODE == 1 ? D : RHO;
    constexpr int W = (FAST % VEC == 0) ? VEC : 1;  // outputs per lane (one 16-byte store)
    constexpr int NO = TILE / W;
    const R sc = (R)d.scale;
    const uint64_t pol = policy_evict_first();
    if constexpr (MODE == 1 && !MASK && NT % (D * F / W) == 0) {
      // each thread owns fixed (f, s..s+W-1) and walks m with constant strides
      constexpr int PER_M = D * F / W;  // outputs per m-plane
      constexpr int MSTEP = NT / PER_M;
      const int o = tx() * W;
      const int s0 = o % D, f = (o / D) % F, m0 = o / (D * F);
      V* ptr = dst + f * d.of + s0 * d.os + (int64_t)m0 * d.om;
      const int64_t pstep = (int64_t)MSTEP * d.om;
      const int ib = sidx(f, s0, m0);
#pragma unroll 4
      for (int it = 0; it < RHO / MSTEP; ++it) {
        V y[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          y[w] = sm[ib + it * MSTEP * D * PADF + w * PADF];
          if constexpr (CS) y[w] = mk(y[w].x * sc, -y[w].y * sc);
        }
        if constexpr (W == 2)
          st_hint(reinterpret_cast<float4*>(ptr), pack(y[0], y[W - 1]), pol);
        else
          st_hint(ptr, y[0], pol);
        ptr += pstep;
      }
      return;
    }
#pragma unroll 4
    for (int o0 = tx(); o0 < NO; o0 += NT) {
      const int o = o0 * W;
      int f, s, m;
      if constexpr (MODE == 1) {
        s = o % D;
        f = (o / D) % F;
        m = o / (D * F);
      } else {
        m = o % RHO;
        s = (o / RHO) % D;
        f = o / (RHO * D);
      }
      if (MASK && grp * d.cg + s * d.cs + f >= d.ncols) continue;
      V y[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        y[w] = MODE == 1 ? sm[sidx(f, s + w, m)] : sm[sidx(f, s, m + w)];
        if constexpr (CS) y[w] = mk(y[w].x * sc, -y[w].y * sc);
      }
      V* ptr = dst + f * d.of + s * d.os + (int64_t)m * d.om;
      if constexpr (W == 2)
        st_hint(reinterpret_cast<float4*>(ptr), pack(y[0], y[W - 1]), pol);
      else
        st_hint(ptr, y[0], pol);
    }
  }

  __device__ __forceinline__ static void store(const SubDesc& d, const PassArgs& p, int64_t grp, int task,
                                               int slot, const V* v, V* sm) {
    V* dst = d.out_staging ? (V*)p.staging + slot * p.slot_elems + task * d.ot
                           : (V*)p.out + grp * d.og + task * d.ot;
    const bool cs = d.conj_out;
    if (d.store_mode == 0) {
      if (cs)
        store_direct<true>(d, dst, grp, v);
      else
        store_direct<false>(d, dst, grp, v);
    } else if (d.store_mode == 1) {
      if (cs)
        store_transposed<true, 1>(d, dst, grp, v, sm);
      else
        store_transposed<false, 1>(d, dst, grp, v, sm);
    } else {
      if (cs)
        store_transposed<true, 2>(d, dst, grp, v, sm);
      else
        store_transposed<false, 2>(d, dst, grp, v, sm);
    }
  }

  __device__ __forceinline__ static const V* source(const SubDesc& d, const PassArgs& p, int64_t grp, int task,
                                                     int slot) {
    return d.in_staging ? (const V*)p.staging + (int64_t)slot * p.slot_elems + task * d.it
                        : (const V*)p.in + grp * d.ig + task * d.it;
  }

  __device__ __forceinline__ static void load_any(const SubDesc& d, const V* src, int64_t grp, V* v,
                                                  bool& nonfinite) {
    if (d.conj_in) {
      if (d.check_finite)
        load<true, true>(d, src, grp, v, nonfinite);
      else
        load<true, false>(d, src, grp, v, nonfinite);
    } else if (d.check_finite) {
      load<false, true>(d, src, grp, v, nonfinite);
    } else {
      load<false, false>(d, src, grp, v, nonfinite);
    }
  }

  // Everything after the load: DIT twiddle, radix stages, store.  For a tile
  // that read the staging ring (`release` set), the consumed rows are
  // discarded and the slot released once stage 0 has consumed the registers.
  __device__ __forceinline__ static void process(const SubDesc& d, const PassArgs& p, int64_t grp, int task,
                                                 int slot, V* v, V* sm, const V* tw, int32_t* release,
                                                 const V* src) {
    if (d.tw_mod) twiddle(d, grp, task, v);
    if (release != nullptr) {
      stage_compute<0>(v, tw);
      discard_loaded(d, src);
      tsync();
      if (tx() == 0) {
        __threadfence();
        atomicAdd(release, 1);
      }
      if constexpr (NST > 1) {
        stage_write<0>(v, sm);
        tsync();
        stages<1>(v, sm, tw);
      }
    } else {
      stages<0>(v, sm, tw);
    }
    store(d, p, grp, task, slot, v, sm);
  }

  // One tile: load (+conj, +finite check, +DIT twiddle), RHO-point DFTs, store.
  __device__ static void run(const SubDesc& d, const PassArgs& p, int64_t grp, int task, int slot, V* sm,
                             const V* tw, bool& nonfinite, int32_t* release = nullptr) {
    V v[E];
    const V* src = source(d, p, grp, task, slot);
    load_any(d, src, grp, v, nonfinite);
    process(d, p, grp, task, slot, v, sm, tw, release, src);
  }

  __device__ __forceinline__ static void fixup(const SubDesc& d, V* v, bool& nonfinite) {
    const bool cj = d.conj_in, ck = d.check_finite;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (cj) v[i].y = -v[i].y;
      if (ck) nonfinite |= !(isfinite(v[i].x) && isfinite(v[i].y));
    }
  }

  // Warp-specialised variant: the producer warp has copied the tile's 128-byte
  // rows into `buf` (padded rows, mbarrier-signalled); `buf` then doubles as
  // the exchange buffer.  If `release` is set the rows came from the L2
  // staging ring at `stg`: they are discarded (no write-back) and the slot is
  // released to the producers of the next group.
  __device__ static void run_smem(const SubDesc& d, const PassArgs& p, int64_t grp, int task, int slot, V* buf,
                                  const V* tw, bool& nonfinite, int32_t* release, const V* stg) {
    V v[E];
    if (release != nullptr) {
      for (int r = tx(); r < D * RHO; r += NT) l2_discard(stg + (r % D) * d.is + (int64_t)(r / D) * d.im);
    }
    stage_read<0, SWZ>(v, buf);
    tsync();  // every tile thread has its stage-0 data (and issued its discards)
    if (release != nullptr && tx() == 0) red_release_add(release, 1);
    if (d.conj_in || d.check_finite) fixup(d, v, nonfinite);
    if (d.tw_mod) twiddle(d, grp, task, v);
    stage_compute<0>(v, tw);
    if constexpr (NST > 1) {
      stage_write<0>(v, buf);
      tsync();
      stages<1>(v, buf, tw);
    }
    store(d, p, grp, task, slot, v, buf);
  }
};

// Empty B-tile marker for direct (un-staged) passes.
struct NoTile {
  static constexpr int SMEM_ELEMS = 0, RHO = 0, NT = 0;
};

__device__ __forceinline__ void wait_at_least(const int32_t* ctr, int32_t need) {
  if (threadIdx.x == 0) {
    while (*(volatile const int32_t*)ctr < need) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

// Task order of a staged pass: A(0..lag-1), then pairs [B(g-lag), A(g)], then
// the remaining B.  Every dependency (B(g) on A(g), A(g) on the slot released
// by B(g-nslots)) points to an earlier task.
__device__ __forceinline__ void decode_task(const PassArgs& p, int64_t pos, bool& isB, int64_t& grp,
                                            int64_t& sub) {
  const int64_t G = p.ngroups, L = p.lag, TAn = p.a.ntasks, TBn = p.b.ntasks;
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
}

// Persistent pass kernel: CTAs pull tasks from one global counter in a fixed
// order (A(0..lag-1), then B(g-lag), A(g) pairs, then the tail of B), which
// makes every wait target a task that an already-running CTA owns.
// occupancy target: small (32 KB) tiles run 4 CTAs per SM, 64 KB tiles 2
template <class TA> constexpr int min_blocks() {
  return TA::NT >= 512 ? 1 : (TA::TILE * (int)sizeof(typename TA::V) <= 32768 ? 4 : 2);
}

template <typename R, class TA, class TB>
__global__ void __launch_bounds__(TA::NT, min_blocks<TA>()) pass_kernel(const __grid_constant__ PassArgs p) {
  using V = typename CT<R>::V;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int SM_ELEMS = TA::SMEM_ELEMS > TB::SMEM_ELEMS ? TA::SMEM_ELEMS : TB::SMEM_ELEMS;
  V* sm = reinterpret_cast<V*>(smem_raw);
  V* twA = sm + SM_ELEMS;
  V* twB = twA + TA::RHO;
  __shared__ long long s_pos, s_grp;
  __shared__ int s_sub, s_slot, s_isB;
  TA::build_table(twA);
  if constexpr (TB::RHO > 0) TB::build_table(twB);
  bool nonfinite = false;
  // thread 0 claims and decodes tasks (one 64-bit division per task, not per thread)
  auto publish = [&](unsigned long long pos) {
    s_pos = (long long)pos;
    if ((int64_t)pos >= p.total_tasks) return;
    if constexpr (TB::RHO == 0) {
      s_isB = 0;
      s_grp = (long long)(pos / (unsigned long long)p.a.ntasks);
      s_sub = (int)(pos % (unsigned long long)p.a.ntasks);
      s_slot = 0;
    } else {
      bool isB;
      int64_t grp, sub;
      decode_task(p, (int64_t)pos, isB, grp, sub);
      s_isB = isB;
      s_grp = grp;
      s_sub = (int)sub;
      s_slot = (int)(grp % p.nslots);
    }
  };
  if (threadIdx.x == 0) publish(atomicAdd(p.task_counter, 1ull));
  for (;;) {
    __syncthreads();
    const long long pos = s_pos;
    if (pos >= p.total_tasks) break;
    const bool isB = s_isB;
    const int64_t grp = s_grp;
    const int sub = s_sub, slot = s_slot;
    // claim the next task now; its latency hides behind this task's work
    // (deadlock-free: the smallest unfinished task is always a running one)
    unsigned long long next = 0;
    if (threadIdx.x == 0) next = atomicAdd(p.task_counter, 1ull);
    if constexpr (TB::RHO == 0) {
      TA::run(p.a, p, grp, sub, slot, sm, twA, nonfinite);
      __syncthreads();
    } else {
      if (!isB) {
        if (grp >= p.nslots && !p.nowait) wait_at_least(p.doneB + (grp - p.nslots), p.b.ntasks);
        TA::run(p.a, p, grp, sub, slot, sm, twA, nonfinite);
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(p.doneA + grp, 1);
        }
      } else {
        if (!p.nowait) wait_at_least(p.doneA + grp, p.a.ntasks);
        TB::run(p.b, p, grp, sub, slot, sm, twB, nonfinite, p.doneB + grp);
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) publish(next);
  }
  if (__syncthreads_or(nonfinite) && threadIdx.x == 0) atomicOr(p.flag, 1);
}

// Warp-specialised staged pass (persistent).
//   warp 0 (producer) owns every global synchronisation: it claims tasks in
//     order, waits for their producers, issues ONE TMA tensor copy per tile
//     into an NBUF-deep ring of shared-memory buffers, and -- when a buffer
//     comes back -- retires the task that used it: B tiles discard their
//     consumed staging lines and release the ring slot, A tiles publish their
//     group counter (release reduction).
//   warps 1.. (consumers) only compute: wait on the buffer's `full`
//     mbarrier, run the tile (the buffer doubles as the exchange buffer,
//     named barrier 1), store, arrive on `empty`.
template <typename R, class TA, class TB, int NBUF = 2>
__global__ void __launch_bounds__(TA::NT + 32, (TA::TILE * (int)sizeof(typename TA::V) <= 32768 ? 2 : 1))
    staged_kernel(const __grid_constant__ PassArgs p) {
  using V = typename CT<R>::V;
  static_assert(TA::NT == TB::NT && TA::TOFF == 32 && TB::TOFF == 32, "consumer warps follow warp 0");
  static_assert(TA::SWZ && TB::SWZ, "TMA tiles land 128B-swizzled");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int BUF = TA::SMEM_ELEMS > TB::SMEM_ELEMS ? TA::SMEM_ELEMS : TB::SMEM_ELEMS;
  static_assert((BUF * sizeof(V)) % 1024 == 0, "swizzled buffers stay 1024-byte aligned");
  V* bufs = reinterpret_cast<V*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  V* twA = bufs + NBUF * BUF;
  V* twB = twA + TA::RHO;
  __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF];
  __shared__ long long task_of[NBUF], task_grp[NBUF];
  __shared__ int task_sub[NBUF], task_slot[NBUF], task_isB[NBUF];
  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], TA::NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  TA::build_table(twA);
  TB::build_table(twB);
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    const uint64_t pol = policy_evict_first();
    // retire the task that last used buffer b (its consumers are done)
    auto retire = [&](int b) {
      if (task_of[b] < 0) return;
      const int64_t grp = task_grp[b];
      if (task_isB[b]) {
        const V* stg = (const V*)p.staging + (int64_t)task_slot[b] * p.slot_elems + (int64_t)task_sub[b] * p.b.it;
        for (int r = lane; r < TB::D * TB::RHO; r += 32)
          l2_discard(stg + (r % TB::D) * p.b.is + (int64_t)(r / TB::D) * p.b.im);
        __syncwarp();
        if (lane == 0) red_release_add(p.doneB + grp, 1);
      } else if (lane == 0) {
        red_release_add(p.doneA + grp, 1);
      }
      task_of[b] = -1;
    };
    for (int i = 0; i < NBUF; ++i) task_of[i] = -1;
    // per-buffer counts of issued and retired tasks (warp-uniform)
    int used[NBUF], retired[NBUF];
#pragma unroll
    for (int i = 0; i < NBUF; ++i) used[i] = retired[i] = 0;
    auto retire_one = [&](int b) {
      mbar_wait_dbg(&empty[b], (uint32_t)(retired[b] & 1), 1, b, retired[b]);
      retire(b);
      ++retired[b];
    };
    // retire every outstanding buffer, oldest first (this CTA then holds no
    // unfinished task, so a blocking dependency wait cannot deadlock)
    auto drain = [&](int64_t k) {
      for (int64_t j = k - NBUF + 1; j < k; ++j) {
        if (j < 0) continue;
        const int bb = (int)(j % NBUF);
        if (retired[bb] < used[bb]) retire_one(bb);
      }
    };
    int64_t k = 0;
    for (;; ++k) {
      const int b = (int)(k % NBUF);
      if (retired[b] < used[b]) retire_one(b);
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(p.task_counter, 1ull);
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if ((int64_t)pos >= p.total_tasks) {
        if (lane == 0) {
          task_of[b] = -2;  // end marker for the consumers (never retired)
          mbar_arrive(&full[b]);
        }
        break;
      }
      bool isB;
      int64_t grp, sub;
      decode_task(p, (int64_t)pos, isB, grp, sub);
      const int32_t* ctr = isB ? p.doneA + grp : (grp >= p.nslots ? p.doneB + (grp - p.nslots) : nullptr);
      const int32_t need = isB ? p.a.ntasks : p.b.ntasks;
      if (ctr != nullptr && !p.nowait) {
        int ok = 0;
        if (lane == 0) ok = ld_acquire(ctr) >= need;
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) {
          drain(k);
          if (lane == 0)
          {
            long long n = 0;
            while (ld_acquire(ctr) < need) {
              __nanosleep(32);
              if (++n == (1ll << 27)) {
                printf("EFFT STUCK dep cta=%d pos=%lld isB=%d grp=%lld need=%d have=%d\n", blockIdx.x,
                       (long long)pos, (int)isB, (long long)grp, need, ld_acquire(ctr));
                __trap();
              }
            }
          }
          __syncwarp();
        }
      }
      if (lane == 0) {
        fence_proxy_async();
        task_of[b] = (long long)pos;
        task_grp[b] = grp;
        task_sub[b] = (int)sub;
        task_slot[b] = (int)(grp % p.nslots);
        task_isB[b] = isB;
        V* dst = bufs + b * BUF;
        if (!isB) {
          constexpr int W = (int)sizeof(V) / 8;
          constexpr int BOX = TA::RHO > 256 ? TA::RHO / 2 : TA::RHO;
          mbar_arrive_tx(&full[b], (uint32_t)(TA::D * TA::RHO * 128));
#pragma unroll
          for (int h = 0; h < TA::RHO / BOX; ++h)
            tma_load_3d(dst + h * BOX * TA::D * TA::F, &p.tmA, (int)(grp * TA::F * W), (int)(sub * TA::D),
                        h * BOX, &full[b], pol);
        } else {
          constexpr int BOX = TB::RHO > 256 ? TB::RHO / 2 : TB::RHO;
          mbar_arrive_tx(&full[b], (uint32_t)(TB::D * TB::RHO * 128));
#pragma unroll
          for (int h = 0; h < TB::RHO / BOX; ++h)
            tma_load_4d(dst + h * BOX * TB::D * TB::F, &p.tmB, 0, (int)(sub * TB::D), h * BOX, task_slot[b],
                        &full[b], pol);
        }
      }
      __syncwarp();
      ++used[b];
    }
    drain(k);  // retire the tasks still holding buffers (buffer k%NBUF holds the end marker)
  } else {
    bool nonfinite = false;
    for (int64_t k = 0;; ++k) {
      const int b = (int)(k % NBUF);
      mbar_wait_dbg(&full[b], (uint32_t)((k / NBUF) & 1), 2, b, k);
      const long long pos = task_of[b];
      if (pos == -2) break;
      const bool isB = task_isB[b];
      const int64_t grp = task_grp[b];
      const int sub = task_sub[b], slot = task_slot[b];
      V* buf = bufs + b * BUF;
      if (!isB)
        TA::run_smem(p.a, p, grp, sub, slot, buf, twA, nonfinite, nullptr, nullptr);
      else
        TB::run_smem(p.b, p, grp, sub, slot, buf, twB, nonfinite, nullptr, nullptr);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    if (nonfinite) atomicOr(p.flag, 1);
  }
}

// ----------------------------------------------------------------------------
// Block permutations used by the sharded (multi-GPU) six-step: pack/unpack of
// all-to-all chunks.  Elements are opaque 8- or 16-byte words (VT).
// ----------------------------------------------------------------------------
// out[b][a][c] = in[a][b][c], shapes (n0, n1, n2): the two outer dims swap, the
// contiguous inner dim is copied with 16-byte vectors.
template <typename W>
__global__ void swap01_kernel(const W* __restrict__ in, W* __restrict__ out, int64_t n0, int64_t n1, int64_t n2) {
  const int64_t total = n0 * n1 * n2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % n2, ab = i / n2, b = ab % n1, a = ab / n1;
    out[(b * n0 + a) * n2 + c] = in[i];
  }
}
// out[a][c][b] = in[a][b][c], shapes (n0, n1, n2): a batched 2D transpose
// through a padded 32x33 shared-memory tile.
template <typename W>
__global__ void swap12_kernel(const W* __restrict__ in, W* __restrict__ out, int64_t n1, int64_t n2) {
  __shared__ W t[32][33];
  const int64_t a = blockIdx.z;
  const int64_t b0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const W* src = in + a * n1 * n2;
  W* dst = out + a * n1 * n2;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t b = b0 + y, c = c0 + threadIdx.x;
    if (b < n1 && c < n2) t[y][threadIdx.x] = src[b * n2 + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, b = b0 + threadIdx.x;
    if (b < n1 && c < n2) dst[c * n1 + b] = t[threadIdx.x][y];
  }
}

}  // namespace efft

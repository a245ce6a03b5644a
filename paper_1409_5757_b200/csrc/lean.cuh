// lean.cuh -- host-side interface of the lean staged passes (lean.cu).
//
// The lean path runs the large power-of-two complex64 transforms
// (N = R1 * R2, R = 256 * rho_b with rho_b in {32, 64, 128, 256}, i.e.
// 2^26 <= N <= 2^32) as two staged passes of one persistent kernel each:
//   pass 1: x[j2 + R2*j1] -> y[k1 + R1*j2] (DFT over j1, the four-step twiddle
//           W_N^(j2*k1) fused into the store, the j2 <-> k1 transpose fused
//           into sub-stage A's register exchange)
//   pass 2: y[k1 + R1*j2] -> X[k1 + R1*k2] in place (DFT over j2)
// Each pass is sub-stage A (256-point DFTs, HBM -> L2 staging ring) and
// sub-stage B (rho_b-point DFTs, ring -> HBM), 4096-element tiles, 256
// threads, 16 elements per thread, four CTAs per SM.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace efft {
namespace lean {

struct Args {
  const float2* src;
  float2* dst;
  float2* stg;
  int64_t LS;          // element stride between successive DFT points in src
  int64_t R;           // DFT length of the pass (256 * RB)
  int64_t N;           // full transform length (four-step twiddle of pass 1)
  int64_t slot_elems;  // 16 * R
  int64_t total;       // ngroups * (ntA + ntB)
  int32_t ngroups, nslots, lag, nt;  // nt = tasks per group and sub-stage (RB)
  unsigned long long* ctr;
  int32_t* doneA;
  int32_t* doneB;
  int32_t* flag;
  const float2* t4;  // pass 1: W_N^(i << 20), W_N^(i << 10), W_N^i, i < 1024 (plan-owned, fp64-built)
  float2 cin;   // (1, +-1): conjugation of the pass input
  float2 cout;  // (s, +-s): conjugation and scale of the pass output
  int32_t check_finite;
  // TMA: A tiles read src as [lane, group, ja, jb]; T1 B tiles read the ring as
  // [kt, ks, ja, j2l, slot] (T0 B tiles are contiguous: one bulk copy)
  alignas(64) CUtensorMap tmA;
  alignas(64) CUtensorMap tmB;
};

struct Pass {
  Args a;
  void (*fn)(Args);
  int grid, nt, smem;
  int rb;
  int64_t counter_ints;  // 2 (task counter) + 2 * ngroups
  const void* tmA_src;   // pointer tmA was encoded for
};

// (Re)encode the A-tile tensor map for a pass input / the B-tile map for the ring.
bool encode_src(Pass& p, const void* src);
bool encode_stg(Pass& p, void* stg, int nslots_total);

// Fills p[0], p[1] for n (complex64) or returns false when the lean path does
// not cover n.  Also reports the staging elements the two passes need.
// Writes the pass-1 four-step tables (3 x 1024 complex64) for transform length n.
void build_tables(float2* t4, int64_t n, cudaStream_t s);

bool plan(int64_t n, int inverse, bool scale_inverse, bool check_finite, int num_sms, Pass p[2],
          int64_t* staging_elems, int* err_cuda);

}  // namespace lean
}  // namespace efft

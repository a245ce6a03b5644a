// tpass.cuh -- host-side interface of the TMA-pipelined staged passes (tpass.cu).
//
// Same four-step decomposition as the lean passes (lean.cuh), re-tiled for the
// B200 memory system as measured by tools/skel_bench.cu:
//   * a column group is F = 32 complex64 columns, so every HBM access is a
//     256-byte segment (128-byte segments cap a strided pass at 4.4 TB/s,
//     256-byte ones reach 5.9 TB/s);
//   * every tile (64 KB: 256 rows x 32 columns, or 128 x 64 from the ring) is
//     fetched by ONE TMA instruction into a shared-memory landing buffer while
//     the CTA computes the previous tile (the LDG gather of the lean kernels is
//     request-rate bound);
//   * twiddles are computed per tile in fp64 from exact integer exponents
//     (no global table).
// Pass 1: x[j2 + R2 j1] -> y[k1 + R1 j2] W_N^(j2 k1); pass 2: y -> X[k1 + R1 k2]
// in place.  R = 256 * 128 per pass (N = 2^30, configuration C3).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace efft {
namespace tpass {

struct Args {
  CUtensorMap mapA;  // pass input: dims {LS (column), RB (ja), RA (jb)}, box {32, 1, 256}
  CUtensorMap mapB;  // pass 1 ring: dims {256 (ka), RB (ja), 32 (column), nslots}, box {64, RB, 1, 1}
  const void* src;
  void* dst;
  void* stg;
  int64_t LS;          // element stride between successive DFT points in src
  int64_t R;           // DFT length of the pass (256 * RB)
  int64_t N;           // full transform length (pass-1 twiddle)
  int64_t slot_elems;  // 32 * R: one column group
  int64_t total;       // ngroups * (ntA + ntB) tasks
  int32_t ngroups, nslots, lag;
  int32_t ntA, ntB;
  unsigned long long* ctr;
  int32_t* doneA;
  int32_t* doneB;
  int32_t* flag;
  double2 cin;   // (1, +-1): conjugation of the pass input
  double2 cout;  // (s, +-s): conjugation and scale of the pass output
  int32_t check_finite;
  unsigned long long* prof;  // diagnostics (EFFT_TP_PROF): [2 tile kinds][8 warps][6 phases] cycle sums
};

struct Pass {
  Args a;
  void (*fn)(Args);
  void (*fn_prof)(Args);  // the same kernel with phase timing (EFFT_TP_PROF)
  int grid, nt, smem;
  int rb;
  int64_t counter_ints;  // 2 (task counter) + 2 * ngroups
  const void* mapA_ptr;  // pointer mapA was encoded for
};

// Fills p[0], p[1] for n or returns false when the TMA path does not cover n
// (err_cuda set when a CUDA call failed).  Reports the staging elements needed.
bool plan(int64_t n, int c128, int inverse, bool check_finite, int num_sms, Pass p[2], int64_t* staging_elems,
          int* err_cuda);
// (Re-)encode pass p's input map for `src` (pass 0: d_in, pass 1: d_out); 0 on success.
int encode_input(Pass& p, int pass_index, const void* src);
// Encode the ring map of pass 1 once the staging ring is allocated; 0 on success.
int encode_ring(Pass& p, void* staging);

}  // namespace tpass
}  // namespace efft

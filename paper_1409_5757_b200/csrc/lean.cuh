// lean.cuh -- host-side interface of the lean staged passes (lean.cu).
//
// The lean path runs the large power-of-two transforms (complex64 and
// complex128, N = R1 * R2 with R = rho_a * rho_b, rho_a = 256 (or 192 / 160 /
// 224 in pass 2 for N = 3 / 5 / 7 * 2^k), rho_b in {32, 64, 128, 256} (also
// 16 for complex64): 2^26 (2^24 for complex64) <= N <= 2^32 and the M * 2^k
// families from about 2^24 to 2^30 points) as two staged passes of one persistent kernel each:
//   pass 1: x[j2 + R2*j1] -> y[k1 + R1*j2] (DFT over j1, the four-step twiddle
//           W_N^(j2*k1) fused into the store, the j2 <-> k1 transpose fused
//           into sub-stage A's register exchange)
//   pass 2: y[k1 + R1*j2] -> X[k1 + R1*k2] in place (DFT over j2)
// Each pass is sub-stage A (rho_a-point DFTs, HBM -> L2 staging ring) and
// sub-stage B (rho_b-point DFTs, ring -> HBM); 32 KB tiles, 16 elements per
// thread, four CTAs per SM.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace efft {
namespace lean {

struct Args {
  CUtensorMap mapA;    // prefetching pair kernel: the pass input, box {16, 1, 256}, 128B swizzle
  CUtensorMap mapB;    // prefetching pair kernel, transposing pass: the staging ring
  const void* src;
  void* dst;
  void* stg;
  int64_t LS;          // element stride between successive DFT points in src
  int64_t R;           // DFT length of the pass (256 * RB)
  int64_t N;           // full transform length (four-step twiddle of pass 1)
  int64_t j2off;       // pass 1: global index of the first column (sharded ranks; 0 otherwise)
  int32_t obl;         // pass 1: 0 = transposed output y[k1 + R j2]; else log2 L1 of the blocked
                       //   layout [k1 / L1][j2][k1 % L1] (sharded NCCL path)
  int64_t slot_elems;  // F * R: one column group
  int64_t total;       // ngroups * (ntA + ntB) tasks
  int32_t ngroups, nslots, lag;
  int32_t wg;          // adjacent column groups interleaved in the claim order (lag counts W-group blocks)
  int32_t ntA, ntB;    // tasks per group: A (RB, one per ja), B (RA * RB / 256)
  unsigned long long* ctr;
  int32_t* doneA;
  int32_t* doneB;
  int32_t* flag;
  double2 cin;   // (1, +-1): conjugation of the pass input
  double2 cout;  // (s, +-s): conjugation and scale of the pass output
  int32_t check_finite;
  int32_t abl;   // dev ablation bits of the pipelined kernel (EFFT_PIPE_ABL; 0 in production)
};

struct Pass {
  Args a;
  void (*fn)(Args);
  int grid, nt, smem;
  int ra, rb;
  bool wide = false;  // 32-column groups (lean_wide)
  bool pf = false;    // prefetching pair kernel (TMA landing buffer): needs the tensor maps
  bool pipe = false;  // pipelined pair kernel (producer warp, two TMA buffers)
  const void* mapA_ptr = nullptr;
  int64_t counter_ints;  // 2 (task counter) + 2 * ngroups
};

// Fills p[0], p[1] for n or returns false when the lean path does not cover n
// (err_cuda set when a CUDA call failed).  Reports the staging elements needed.
bool plan(int64_t n, int c128, int inverse, bool scale_inverse, bool check_finite, int num_sms, Pass p[2],
          int64_t* staging_elems, int* err_cuda);

// Six-step over G ranks (efft_execute_sharded): N = N1 N2, G | N1 / F and
// G | N2 / F.  Rank q's local steps are the same two passes on its blocks:
//   pass 1: B_q[n1][c] (N1 x L2, global column q L2 + c) -> Y'_q[c][k1] with
//           W_N^((q L2 + c) k1) fused into the transposing store;
//   pass 2: T_q[n2][k1'] (N2 x L1) -> X_q[k2][k1'] in place (inverse: 1/N).
bool split_sharded(int64_t n, int G, int c128, int64_t* N1, int64_t* N2);
// prefetching pair kernel: (re-)encode the input map for src; encode the ring map (T1); 0 = ok
int encode_input(Pass& p, const void* src);
int encode_ring(Pass& p, void* staging);
bool plan_sharded(int64_t n, int G, int rank, int c128, int inverse, bool check_finite, int num_sms, Pass p[2],
                  int64_t* staging_elems, int* err_cuda, bool blocked = false, int chunks = 1);
// columns per lane group (one 128-byte line; 32 for the wide complex64 kernel): chunk widths must be multiples
int lanes(int c128);

}  // namespace lean
}  // namespace efft

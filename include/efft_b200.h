/*
 * efft_b200.h -- C ABI of the B200 large-1D-FFT library (libefft_b200.so).
 *
 * Plain pointers and sizes only; no C++ exception crosses this boundary and no
 * torch type appears in a signature.  Every function returns an int status
 * (EFFT_OK == 0); efft_last_error() gives a thread-local message.
 *
 * Each entry point replaces a reference interface of the Python package
 * /root/reference/pkg/src/efft (cited file:line):
 *
 *   efft_plan_create      <- plan_create(n, splits, workers, test_mode, ...)   core.py:63-111
 *                            + handle_create(plan) buffer/state set-up         core.py:126-144, 184-186
 *   efft_execute          <- run_transform(handle) / TransformHandle.run()     recombine.py:298-308, core.py:166-170
 *                            (device buffers, enqueued on the caller's stream)
 *   efft_execute_host     <- the same call with host buffers: H2D copy, the two
 *                            passes, D2H copy (what `handle.data[:] = x;
 *                            run_transform(h); h.result` does end to end)
 *   efft_plan_destroy     <- TransformHandle.close()                          core.py:172-174
 *   efft_nonfinite_seen   <- scatter()'s non-finite input check               scatter.py:38-39
 *   efft_plan_create_columns, efft_permute_swap01/12
 *                         <- one recursion level of process_and_reassemble
 *                            (recombine.py:263-295) as a batched column pass +
 *                            the all-to-all packing of the sharded six-step
 *   efft_last_error       <- the exception message of errors.py:4-45
 *
 * Status codes map 1:1 onto the reference exception classes (errors.py).
 */
#ifndef EFFT_B200_H
#define EFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EFFT_OK 0
#define EFFT_ERR_INVALID_ARG 1    /* ValueError                core.py:78-85        */
#define EFFT_ERR_SPLITS_TOO_LARGE 2 /* SplitsTooLarge          core.py:87-89        */
#define EFFT_ERR_SIZE_CONSTRAINT 3 /* SizeConstraintViolation core.py:90-94        */
#define EFFT_ERR_UNSUPPORTED_SIZE 4 /* BinsizeNotPowerOfTwo    core.py:95-100 (here: N not M*2^t, M in {1,3,5,7}) */
#define EFFT_ERR_ALLOC 5          /* AllocationFailure         memory.py:51-54      */
#define EFFT_ERR_SIZE_MISMATCH 6  /* SizeMismatch              scatter.py:34-37     */
#define EFFT_ERR_NONFINITE 7      /* ValueError (non-finite)   scatter.py:38-39     */
#define EFFT_ERR_CUDA 8           /* CUDA runtime failure                           */
#define EFFT_ERR_NCCL 9           /* collective failure (sharded path)              */

#define EFFT_C64 1   /* complex64  (float2)  */
#define EFFT_C128 2  /* complex128 (double2) */
#define EFFT_R32 3   /* real float32 input, reference PERM-packed output
                        [R_0, R_{n/2}, R_1, I_1, ...] (core.py:10-15), forward only */

#define EFFT_FORWARD (-1) /* unnormalised exp(-2 pi i k n / N) (oracle.py:1-8)  */
#define EFFT_INVERSE (+1) /* exp(+2 pi i k n / N), scaled by 1/N               */

/* flags for efft_plan_create */
#define EFFT_FLAG_CHECK_FINITE 0x1u  /* detect non-finite input inside pass 1 */
#define EFFT_FLAG_SCALE_INVERSE 0x2u /* column plans: scale the inverse by 1/len */

typedef struct efft_plan_s *efft_plan_t;

/* Plan one forward or inverse transform of n complex elements on `device`.
 * n must be M*2^t with M in {1,3,5,7}; allocates the staging ring and counters.
 * The input buffer passed to efft_execute is never written; the output buffer
 * doubles as the pass-1 intermediate (out-of-place, two device arrays). */
int efft_plan_create(efft_plan_t *plan, int64_t n, int dtype, int direction, int device,
                     uint32_t flags);

/* Human-readable decomposition (passes, radices, tiles, grid). */
int efft_plan_describe(efft_plan_t plan, char *buf, size_t len);

/* Device workspace owned by the plan (staging ring + counters), bytes. */
int efft_plan_workspace_bytes(efft_plan_t plan, size_t *bytes);

/* Number of kernel launches one efft_execute enqueues. */
int efft_plan_launches(efft_plan_t plan, int *launches);

/* Enqueue the transform on `stream` (cudaStream_t, NULL = legacy default).
 * d_in: n elements (read only); d_out: n elements.  Asynchronous. */
int efft_execute(efft_plan_t plan, const void *d_in, void *d_out, void *stream);

/* End-to-end call with HOST buffers (pinned or pageable): copies h_in to a
 * device input, runs efft_execute, copies the result to h_out and
 * synchronises the stream.  The device in/out pair is one per-device pool
 * shared by all plans (grown on demand, serialised by a lock), so a forward
 * and an inverse plan of the same size need one pair between them. */
int efft_execute_host(efft_plan_t plan, const void *h_in, void *h_out, void *stream);

/* `count` end-to-end transforms with host buffers (h_in[k] -> h_out[k]),
 * pipelined: transform k+1's host-to-device copy runs on an internal copy
 * stream while transform k computes and copies back on `stream`, so both PCIe
 * directions are busy at once (two device in/out pairs from the per-device
 * pool, kept for later calls; one at a time when the second pair does not fit).
 * Returns after the last copy-back has completed.  Transform k+1's input is
 * read once transform k-1's output has landed, so h_in[j] must not alias any
 * h_out[i] with i >= j - 1 (chained transforms: issue them as separate calls). */
int efft_execute_host_batch(efft_plan_t plan, const void *const *h_in, void *const *h_out, int count,
                            void *stream);

/* Out-of-core transform of a HOST array larger than HBM (the
 * paper's "enormous" N, reference bench.py:115-126 reads binary32 arrays from
 * disk): N = N1 N2 four-step over host memory with at most about
 * `device_bytes` of device buffers (two streams x two buffers), strided DMA
 * straight from / to h_in and h_out (page-locked for the call), block k+1's
 * copies overlapping block k's.  h_out doubles as the intermediate; h_in is
 * not modified (read-only memory, e.g. a read-only file mapping, is read
 * through pinned staging buffers); they must not overlap.  N = M 2^t, M in {1,3,5,7},
 * N1, N2 <= 2^17.  Synchronous.  Inverse scaled by 1/N with
 * EFFT_FLAG_SCALE_INVERSE. */
int efft_execute_outofcore(int64_t n, int dtype, int direction, int device, uint32_t flags, const void *h_in,
                           void *h_out, size_t device_bytes);
/* The split and block sizes efft_execute_outofcore uses: blocks[0..3] =
 * N1, N2, columns per step-1 block, rows per step-2 block.  Host only. */
int efft_outofcore_blocks(int64_t n, int dtype, size_t device_bytes, int64_t *blocks);

/* Frees the per-device pool of efft_execute_host (it is re-created on demand). */
int efft_release_host_buffers(int device);

/* Returns (synchronising) whether any non-finite input value was seen by
 * executions since the last call, and clears the flag. */
int efft_nonfinite_seen(efft_plan_t plan, int *seen, void *stream);

int efft_plan_destroy(efft_plan_t plan);

/* Per-launch device timing (CUDA events recorded on the execution stream
 * around every kernel the plan launches).  enable = K > 0 keeps the events of
 * the last K executions (a ring; 0 switches timing off and drops them); once
 * those executions have completed, efft_plan_launch_times() fills
 * ms[0..launches-1] with each launch's duration averaged over them. */
int efft_plan_enable_timing(efft_plan_t plan, int enable);
int efft_plan_launch_times(efft_plan_t plan, float *ms, int max_launches);

/* Batched column transform (one HBM pass), the local step of the sharded
 * six-step (reference counterpart: the per-bin leaf + merge work of one
 * recursion level, leaf_dft.py:93-125 / recombine.py:216-260, batched).
 * For every column c < cols of a row-major (len x cols) array:
 *   out[c + k*cols] = sum_r in[c + r*cols] * W_tw^((tw_offset + c) * r) * W_len^(r*k)
 * W_m = exp(direction * 2 pi i / m); tw_mod = 0 disables the twiddle.  Inverse
 * is unscaled unless EFFT_FLAG_SCALE_INVERSE.  len <= 2^17 (one pass); in ==
 * out is allowed. */
int efft_plan_create_columns(efft_plan_t *plan, int64_t len, int64_t cols, int dtype, int direction,
                             int device, int64_t tw_mod, int64_t tw_offset, uint32_t flags);

/* Sharded six-step over G = ngpus devices of ONE process (
 * the reference's only parallelism is the in-process fork-join of
 * parallel.py:34-98 / recombine.py:263-295).  Natural-order block shards:
 * rank q (device devices[q]) holds x[q N/G, (q+1) N/G) in in[q] and receives
 * X[q N/G, (q+1) N/G) in out[q].  N = N1 N2 (efft_sharded_split); per rank two
 * local HBM passes (the lean pass kernels: pass 1 with the four-step twiddle
 * and the transpose fused into its store, pass 2 in place in a plan-owned work
 * array) and three exchanges done as pitched peer copies over NVLink (no
 * pack / unpack / transpose kernels), ordered by cross-device events on the
 * callers' streams (streams[q] on devices[q]).  A device may appear more than
 * once (emulated ranks on one GPU).  Inverse scaled by 1/N.  in[] is not
 * modified. */
int efft_plan_create_sharded(efft_plan_t *plan, int64_t n, int dtype, int direction, int ngpus, const int *devices,
                             uint32_t flags);
int efft_execute_sharded(efft_plan_t plan, const void *const *in, void *const *out, void *const *streams);
int efft_sharded_split(efft_plan_t plan, int64_t *n1, int64_t *n2);

/* The same six-step with one process per GPU (torch.distributed / NCCL
 * drives the exchanges; paper_1409_5757_b200/sharded.py): rank `rank` of
 * `ngpus` on `device`.  Pass 0: B[n1][c] (N1 x L2, global column rank L2 + c)
 * -> Y blocked by destination rank [p][c][k1'] (the all-to-all send buffer) with
 * the four-step twiddle fused; pass 1: T[n2][k1'] (N2 x L1) -> X[k2][k1'] in
 * place (inverse: 1/N).  Asynchronous on `stream`. */
int efft_plan_create_shard_rank(efft_plan_t *plan, int64_t n, int dtype, int direction, int ngpus, int rank,
                                int device, uint32_t flags);
int efft_execute_shard_pass(efft_plan_t plan, int pass, const void *in, void *out, void *stream);

/* Block permutations (all-to-all packing): shapes (n0, n1, n2) of 8- or
 * 16-byte elements.  swap01: out[b][a][c] = in[a][b][c];  swap12:
 * out[a][c][b] = in[a][b][c].  Asynchronous on `stream`; in != out. */
int efft_permute_swap01(const void *in, void *out, int64_t n0, int64_t n1, int64_t n2, int elem_bytes,
                        void *stream);
int efft_permute_swap12(const void *in, void *out, int64_t n0, int64_t n1, int64_t n2, int elem_bytes,
                        void *stream);

const char *efft_last_error(void);
int efft_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EFFT_B200_H */

// efft_capi.cu -- planner, executor and the C ABI (include/efft_b200.h).
//
// Planner (reference counterpart: plan_create, core.py:63-111).  N = M * 2^t,
// M in {1, 3, 5, 7}, is split into at most two Stockham passes N = R1 * R2 (the
// four-step form of the reference's scatter -> leaves -> merges).  A pass whose
// radix fits one tile (<= 512 points, <= 384 with the factor 3) is "direct";
// a larger one is "staged" as R = rho_a * rho_b through the L2 staging ring.
//
// Executor (reference counterpart: run_transform, recombine.py:298-308): one
// memset of the task counters, then one persistent kernel launch per pass,
// all on the caller's stream.  Pass 1 reads `in` and writes `out`; pass 2 runs
// in place on `out` (its tiles read every element they write before writing),
// so the input is preserved (core.py:146-149) with just two device arrays.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "../../include/efft_b200.h"
#include "efft_registry.cuh"
#include "lean.cuh"
#include "tpass.cuh"

using efft::KernelInfo;
using efft::PassArgs;
using efft::SubDesc;

namespace {

// Real-input post-process (reference leaf_dft.py:113-125, in place over the
// half-length complex spectrum Z of the n/2 pairs):
//   F_k = Z_k P_k + conj(Z_{h-k}) Q_k,  P_k = 1/2 - i/2 w^k,  Q_k = 1/2 + i/2 w^k,
//   w = exp(-2 pi i / n); packed as [F_0, F_{n/2}, Re F_1, Im F_1, ...].
// Each pair (k, h-k), 0 < k < h/2, is updated in place by one thread; thread t
// of T handles k = 1 + t + j T, j < SPLIT_K, with w^k from one fp64 sincospi
// base and an fp64 recurrence by w^T (w^(h-k) = -conj(w^k): no second angle).
constexpr int SPLIT_K = 8;
__global__ void real_split_kernel(float2* z, int64_t h, int64_t n) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  if (t == 0) {
    const float2 z0 = z[0];
    z[0] = make_float2(z0.x + z0.y, z0.x - z0.y);
    if (h > 1 && (h & 1) == 0) {  // k = h/2 is self-paired: F = conj(Z)
      const float2 zm = z[h / 2];
      z[h / 2] = make_float2(zm.x, -zm.y);
    }
  }
  int64_t k = 1 + t;
  if (2 * k >= h) return;
  double c, s, cs, ss;
  sincospi(-2.0 * (double)k / (double)n, &s, &c);
  sincospi(-2.0 * (double)T / (double)n, &ss, &cs);
  // F for (zk, zr = Z_{h-k}) with w = (c, s): P = (1/2 + s/2, -c/2), Q = (1/2 - s/2, c/2)
  auto out = [](float2 zk, float2 zr, double c_, double s_) {
    const double pr = 0.5 + 0.5 * s_, pi = -0.5 * c_, qr = 0.5 - 0.5 * s_, qi = 0.5 * c_;
    const double cr = zr.x, ci = -zr.y;  // conj(Z_{h-k})
    return make_float2((float)(zk.x * pr - zk.y * pi + cr * qr - ci * qi),
                       (float)(zk.x * pi + zk.y * pr + cr * qi + ci * qr));
  };
  for (int j = 0; j < SPLIT_K && 2 * k < h; ++j, k += T) {
    const int64_t kk = h - k;
    const float2 a = z[k], b = z[kk];
    z[k] = out(a, b, c, s);
    z[kk] = out(b, a, -c, s);  // w^(h-k) = -conj(w^k)
    const double cn = c * cs - s * ss;
    s = c * ss + s * cs;
    c = cn;
  }
}

thread_local std::string g_err;

// Device in/out pair of efft_execute_host, one per device, shared by all plans.
constexpr int kMaxDevices = 64;
struct HostPool {
  std::mutex mu;
  void* in = nullptr;
  void* out = nullptr;
  size_t bytes = 0;
  // second pair, copy stream and events of efft_execute_host_batch (lazily created)
  void* in2 = nullptr;
  void* out2 = nullptr;
  size_t bytes2 = 0;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};
HostPool& host_pool(int device) {
  static HostPool pools[kMaxDevices];
  return pools[device];
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) return fail(EFFT_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

struct PassPlan {
  const void* tmA_ptr = nullptr;  // pointer the A tensor map was encoded for
  KernelInfo k;
  PassArgs args;
  int grid;
  int64_t radix, rho_a, rho_b;
  int64_t counter_off;  // offset (in int32 units) of this pass's counters
  int64_t counter_len;
  bool staged;
};

}  // namespace

struct efft_plan_s {
  int64_t n;        // complex length the passes run on (n_user / 2 for EFFT_R32)
  int64_t n_user;
  bool real_input = false;
  // batched column plan (efft_plan_create_columns): one pass, column store
  bool columns = false;
  int64_t col_len = 0, col_count = 0, col_tw_mod = 0, col_tw_offset = 0;
  int dtype, direction, device;
  uint32_t flags;
  int npass;
  PassPlan pass[2];
  size_t elem;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  int32_t* counters = nullptr;
  size_t counter_bytes = 0;
  int32_t* flag = nullptr;
  int num_sms = 0;
  bool timing = false;
  // launch boundaries of the last `tcap` executes (4 events each), a ring
  std::vector<cudaEvent_t> tev;
  int tcap = 0;
  long long tcount = 0;
  // lean path (lean.cu): large M * 2^t transforms (both dtypes)
  bool lean = false;
  efft::lean::Pass lp[2];
  // TMA-pipelined path (tpass.cu): complex64 N = 2^30
  bool tp = false;
  efft::tpass::Pass tpp[2];
  // sharded six-step over G devices (efft_plan_create_sharded)
  struct Rank {
    int dev = 0;
    efft::lean::Pass lp[2];
    void* staging = nullptr;
    int32_t* counters = nullptr;
    size_t counter_bytes = 0;
    int32_t* flag = nullptr;
    void* work = nullptr;  // N / G elements
    cudaEvent_t ev = nullptr;
    // overlapped execution (sh_chunks > 1): a second work array (exchange 2 lands
    // while pass 1 still reads `work`), a copy stream, and per-chunk events
    // [exchange 1 in, pass 1, exchange 2 out, pass 2, exchange 3 out]
    void* work2 = nullptr;
    cudaStream_t cs = nullptr, cs2 = nullptr;  // incoming (exchange 1) / outgoing (exchanges 2, 3) copies
    std::vector<cudaEvent_t> cev;
  };
  std::vector<Rank> ranks;
  int sh_chunks = 1;
  int64_t sh_n1 = 0, sh_n2 = 0;
  int sh_rank = 0, sh_world = 0;  // shard-rank plans (efft_plan_create_shard_rank)
};

namespace {

bool factor(int64_t n, int* M, int* t) {
  if (n < 1) return false;
  int tt = 0;
  while ((n & 1) == 0) {
    n >>= 1;
    ++tt;
  }
  if (n != 1 && n != 3 && n != 5 && n != 7) return false;
  *M = (int)n;
  *t = tt;
  return true;
}

bool get_direct(int dtype, int rho, KernelInfo* k) {
  return dtype == EFFT_C64 ? efft::get_direct_kernel_f32(rho, k) : efft::get_direct_kernel_f64(rho, k);
}
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

bool get_staged(int dtype, int ra, int rb, KernelInfo* k) {
  return dtype == EFFT_C64 ? efft::get_staged_kernel_f32(ra, rb, k) : efft::get_staged_kernel_f64(ra, rb, k);
}


// Decide direct vs staged and the sub-radices of one pass of radix R.
bool pick_pass(int dtype, int64_t R, PassPlan* pp) {
  pp->radix = R;
  const bool has3 = (R % 3) == 0, has5 = (R % 5) == 0, has7 = (R % 7) == 0;
  const int64_t dmax = has3 ? 384 : has5 ? 320 : has7 ? 448 : 512;
  if (R <= dmax) {
    pp->staged = false;
    pp->rho_a = R;
    pp->rho_b = 0;
    return get_direct(dtype, (int)R, &pp->k);
  }
  pp->staged = true;
  pp->rho_a = has3 ? 384 : has5 ? 320 : has7 ? 448 : 256;
  pp->rho_b = R / pp->rho_a;
  if (pp->rho_b * pp->rho_a != R || pp->rho_b > 512) return false;
  bool ok;
  ok = get_staged(dtype, (int)pp->rho_a, (int)pp->rho_b, &pp->k);
  if (!ok) return false;
  // A tiles take D_A = tpts/rho_a consecutive u (D_A | rho_b); B tiles cover
  // D_B = tpts/rho_b outputs k1 of the rho_a-point DFTs (D_B | rho_a)
  const int64_t tile = pp->k.tpts;
  const int64_t da = tile / pp->rho_a;
  const int64_t db = pp->k.tpts_b / pp->rho_b;  // outputs k1 per B tile
  return pp->rho_b % da == 0 && pp->rho_b <= pp->k.tpts_b && db > 0 && pp->rho_a % db == 0;
}

SubDesc blank_desc() {
  SubDesc d;
  memset(&d, 0, sizeof d);
  d.scale = 1.0;
  d.ntasks = 1;
  return d;
}

// Fill the descriptors of pass `p` (0-based) of `np` for a Stockham pass with
// radix R and Ns = product of earlier radices.
void describe_pass(efft_plan_s* pl, int p, int np, int64_t R, int64_t Ns) {
  PassPlan& pp = pl->pass[p];
  const int64_t N = pl->n;
  const int64_t C = N / R;                     // columns j of this pass
  const int F = pl->dtype == EFFT_C64 ? 16 : 8;  // 128-byte column runs
  const bool first = p == 0, last = p == np - 1;
  const bool inverse = pl->direction == EFFT_INVERSE;
  PassArgs& a = pp.args;
  memset(&a, 0, sizeof a);
  a.a = blank_desc();
  a.b = blank_desc();
  if (!pp.staged) {
    const int64_t D = pp.k.d_a;
    SubDesc& d = a.a;
    d.ncols = C;
    d.cg = D * F;
    d.cs = F;
    d.ig = D * F;
    d.is = F;
    d.im = C;
    if (Ns == 1) {  // out[j*R + r]: transposed, unit stride along r
      d.og = D * F * R;
      d.of = R;
      d.os = F * R;
      d.om = 1;
      d.store_mode = 2;
    } else {  // Ns == C: out[j + r*C], j-runs
      d.og = D * F;
      d.of = 1;
      d.os = F;
      d.om = C;
      d.store_mode = 0;
      d.tw_mod = N;  // W_N^(j*r)
      d.Ag = D * F;
      d.As = F;
      d.Af = 1;
      d.Cm = 1;
    }
    d.conj_in = first && inverse;
    d.check_finite = first && (pl->flags & EFFT_FLAG_CHECK_FINITE);
    d.conj_out = last && inverse;
    d.scale = (last && inverse) ? 1.0 / (double)N : 1.0;
    d.ntasks = 1;
    a.ngroups = (C + D * F - 1) / (D * F);
    a.total_tasks = a.ngroups;
    a.staged = 0;
    return;
  }
  const int64_t ra = pp.rho_a, rb = pp.rho_b;
  const int64_t DB = pp.k.d_b;
  SubDesc& A = a.a;
  SubDesc& B = a.b;
  // A: rows r = u + t*rb, u = task*DA + s, rho_a-point DFT over t, into staging
  const int64_t DA = pp.k.d_a;
  A.ncols = C;
  A.cg = F;
  A.ig = F;
  A.it = DA * C;
  A.is = C;
  A.im = rb * C;
  if (Ns != 1) {
    A.tw_mod = N;  // W_N^(j*r), j = grp*F + f, r = u + t*rb
    A.Ag = F;
    A.Af = 1;
    A.Ct = DA;
    A.Cs = 1;
    A.Cm = rb;
  }
  A.out_staging = 1;
  A.ot = DA * ra * F;  // staging (u*ra + k1)*F + f
  A.os = ra * F;
  A.om = F;
  A.store_mode = 0;
  A.ntasks = (int32_t)(rb / DA);
  A.conj_in = first && inverse;
  A.check_finite = first && (pl->flags & EFFT_FLAG_CHECK_FINITE);
  // B: k1 = task*DB + s, rho_b-point DFT over u with W_R^(k1*u)
  B.ncols = C;
  B.cg = F;
  B.in_staging = 1;
  B.it = DB * F;
  B.is = F;
  B.im = ra * F;
  B.tw_mod = R;
  B.At = DB;
  B.As = 1;
  B.Cm = 1;
  if (Ns == 1) {  // out[j*R + k1 + ra*k2]: runs along k1 (s)
    B.og = F * R;
    B.of = R;
    B.ot = DB;
    B.os = 1;
    B.om = ra;
    B.store_mode = 1;
  } else {  // out[j + (k1 + ra*k2)*C]
    B.og = F;
    B.of = 1;
    B.ot = DB * C;
    B.os = C;
    B.om = ra * C;
    B.store_mode = 0;
  }
  B.ntasks = (int32_t)(ra / DB);
  B.conj_out = last && inverse;
  B.scale = (last && inverse) ? 1.0 / (double)N : 1.0;
  a.ngroups = C / F;
  a.slot_elems = (int64_t)F * R;
  a.staged = 1;
  a.total_tasks = a.ngroups * (A.ntasks + B.ntasks);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

// TMA map of a staged pass's A tiles over its input: [column (uint64 units), u, t]
int encode_A(efft_plan_s* pl, PassPlan& pp, const void* base) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(EFFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t N = pl->n, R = pp.radix, C = N / R, w = (int64_t)pl->elem / 8;
  const int F = 128 / (int)pl->elem;
  cuuint64_t dims[3] = {(cuuint64_t)(C * w), (cuuint64_t)pp.rho_b, (cuuint64_t)pp.rho_a};
  cuuint64_t strides[2] = {(cuuint64_t)(C * pl->elem), (cuuint64_t)(pp.rho_b * C * pl->elem)};
  cuuint32_t box[3] = {(cuuint32_t)(F * w), (cuuint32_t)pp.k.d_a, (cuuint32_t)(pp.rho_a > 256 ? pp.rho_a / 2 : pp.rho_a)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&pp.args.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EFFT_ERR_CUDA, "tensor map (A) encode failed: %d", (int)r);
  pp.tmA_ptr = base;
  return EFFT_OK;
}

// TMA map of a direct pass's tiles over its input: [f (uint64 units), column group, row]
int encode_D(efft_plan_s* pl, PassPlan& pp, const void* base) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(EFFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t N = pl->n, R = pp.radix, C = N / R, w = (int64_t)pl->elem / 8;
  const int F = 128 / (int)pl->elem;
  cuuint64_t dims[3] = {(cuuint64_t)(F * w), (cuuint64_t)(C / F), (cuuint64_t)R};
  cuuint64_t strides[2] = {(cuuint64_t)(F * pl->elem), (cuuint64_t)(C * pl->elem)};
  cuuint32_t box[3] = {(cuuint32_t)(F * w), (cuuint32_t)pp.k.d_a, (cuuint32_t)(R > 256 ? R / 2 : R)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&pp.args.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EFFT_ERR_CUDA, "tensor map (direct) encode failed: %d", (int)r);
  pp.tmA_ptr = base;
  return EFFT_OK;
}

// TMA map of a staged pass's B tiles over the staging ring: [f, k1, u, slot]
int encode_B(efft_plan_s* pl, PassPlan& pp) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(EFFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t R = pp.radix, w = (int64_t)pl->elem / 8;
  const int F = 128 / (int)pl->elem;
  cuuint64_t dims[4] = {(cuuint64_t)(F * w), (cuuint64_t)pp.rho_a, (cuuint64_t)pp.rho_b, (cuuint64_t)pp.args.nslots};
  cuuint64_t strides[3] = {(cuuint64_t)(F * pl->elem), (cuuint64_t)(pp.rho_a * F * pl->elem),
                           (cuuint64_t)(R * F * pl->elem)};
  cuuint32_t box[4] = {(cuuint32_t)(F * w), (cuuint32_t)pp.k.d_b,
                       (cuuint32_t)(pp.rho_b > 256 ? pp.rho_b / 2 : pp.rho_b), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&pp.args.tmB, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, pl->staging, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EFFT_ERR_CUDA, "tensor map (B) encode failed: %d", (int)r);
  return EFFT_OK;
}

int build_plan(efft_plan_s* pl) {
  int M, t;
  if (pl->columns) {
    if (!factor(pl->col_len, &M, &t) || pl->col_len < 2)
      return fail(EFFT_ERR_UNSUPPORTED_SIZE, "len=%lld is not M*2^t with M in {1,3,5,7}", (long long)pl->col_len);
  } else if (!factor(pl->n, &M, &t) || pl->n < 2)
    return fail(EFFT_ERR_UNSUPPORTED_SIZE,
                "n=%lld is not M*2^t with M in {1,3,5,7} and n >= 2", (long long)pl->n);
  const int dt = pl->dtype;
  if (!pl->columns && env_int("EFFT_LEAN", 1)) {
    int64_t stg = 0;
    int ecuda = 0;
    if (efft::tpass::plan(pl->n, dt == EFFT_C128, pl->direction == EFFT_INVERSE,
                          (pl->flags & EFFT_FLAG_CHECK_FINITE) != 0, pl->num_sms, pl->tpp, &stg, &ecuda)) {
      pl->tp = true;
      pl->npass = 2;
      pl->staging_bytes = (size_t)stg * pl->elem;
      pl->counter_bytes = (size_t)(pl->tpp[0].counter_ints + pl->tpp[1].counter_ints) * 4;
      return EFFT_OK;
    }
    if (ecuda) return fail(EFFT_ERR_CUDA, "TMA pass setup failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (efft::lean::plan(pl->n, dt == EFFT_C128, pl->direction == EFFT_INVERSE, true,
                         (pl->flags & EFFT_FLAG_CHECK_FINITE) != 0, pl->num_sms, pl->lp, &stg, &ecuda)) {
      pl->lean = true;
      pl->npass = 2;
      pl->staging_bytes = (size_t)stg * pl->elem;
      pl->counter_bytes = (size_t)(pl->lp[0].counter_ints + pl->lp[1].counter_ints) * 4;
      return EFFT_OK;
    }
    if (ecuda) return fail(EFFT_ERR_CUDA, "lean pass setup failed: %s", cudaGetErrorString(cudaGetLastError()));
  }
  int64_t R1, R2;
  const int64_t dmax = M == 3 ? 384 : M == 5 ? 320 : M == 7 ? 448 : 512;
  if (pl->columns) {
    pl->npass = 1;
    R1 = pl->col_len;
    R2 = 1;
    PassPlan a;
    if (!pick_pass(dt, R1, &a))
      return fail(EFFT_ERR_UNSUPPORTED_SIZE, "no single-pass kernel for len=%lld", (long long)R1);
    const int F = dt == EFFT_C64 ? 16 : 8;
    if (a.staged && pl->col_count % F)
      return fail(EFFT_ERR_UNSUPPORTED_SIZE, "cols=%lld must be a multiple of %d for len=%lld",
                  (long long)pl->col_count, F, (long long)R1);
  } else if (pl->n <= dmax) {
    pl->npass = 1;
    R1 = pl->n;
    R2 = 1;
  } else {
    pl->npass = 2;
    // Beyond two direct passes (n > dmax^2) the first pass is a direct one of
    // radix M*2^k <= 256 (c128) / 512 (c64) / dmax (M > 1) and the second a
    // staged one: 1.1-1.9x the balanced two-staged split on B200 from 2^21 to
    // 2^25 (tools/split_sizes.py, profiles/r01_split_sizes.txt).  Otherwise a
    // balanced split; the odd factor goes to pass 1.  EFFT_SPLIT_T1 (log2 of
    // pass 1's power of two) overrides both, for experiments.
    const int F2 = dt == EFFT_C64 ? 16 : 8;
    int t1 = env_int("EFFT_SPLIT_T1", -1);
    PassPlan a, b;
    if (t1 < 0 && pl->n > dmax * dmax) {
      const int64_t cap = M == 1 ? (dt == EFFT_C128 ? 256 : 512) : dmax;
      int k = 0;
      while (k < t && ((int64_t)M << (k + 1)) <= cap) ++k;
      const int64_t r1 = (int64_t)M << k, r2 = pl->n / r1;
      if (pick_pass(dt, r1, &a) && !a.staged && pick_pass(dt, r2, &b) && (!b.staged || r1 % F2 == 0)) t1 = k;
    }
    if (t1 < 0 || t1 > t) t1 = t / 2;
    R1 = (int64_t)M << t1;
    R2 = pl->n / R1;
    if (!pick_pass(dt, R1, &a) || !pick_pass(dt, R2, &b)) {
      // shift one power of two between the passes and retry
      bool ok = false;
      for (int d : {-1, 1, -2, 2}) {
        const int tt = t1 + d;
        if (tt < 0 || tt > t) continue;
        R1 = (int64_t)M << tt;
        R2 = pl->n / R1;
        if (pick_pass(dt, R1, &a) && pick_pass(dt, R2, &b)) {
          ok = true;
          break;
        }
      }
      if (!ok) return fail(EFFT_ERR_UNSUPPORTED_SIZE, "no decomposition for n=%lld", (long long)pl->n);
    }
    // staged passes need >= F columns
    const int F = dt == EFFT_C64 ? 16 : 8;
    if ((a.staged && (pl->n / R1) % F) || (b.staged && (pl->n / R2) % F))
      return fail(EFFT_ERR_UNSUPPORTED_SIZE, "n=%lld too small for its decomposition", (long long)pl->n);
  }
  const int64_t radices[2] = {R1, R2};
  int64_t ns = 1;
  int64_t coff = 2;  // int32 units; [0,2) = 64-bit task counter of pass 0
  size_t staging_bytes = 0;
  for (int p = 0; p < pl->npass; ++p) {
    PassPlan& pp = pl->pass[p];
    if (!pick_pass(dt, radices[p], &pp))
      return fail(EFFT_ERR_UNSUPPORTED_SIZE, "no kernel for radix %lld", (long long)radices[p]);
    describe_pass(pl, p, pl->npass, radices[p], pl->columns ? pl->col_count : ns);
    if (pl->columns) {  // column store (Ns = cols), caller-chosen twiddle, unscaled inverse
      SubDesc& d = pp.staged ? pp.args.a : pp.args.a;
      const bool inverse = pl->direction == EFFT_INVERSE;
      SubDesc& last = pp.staged ? pp.args.b : pp.args.a;
      d.tw_mod = pl->col_tw_mod;
      d.A0 = pl->col_tw_offset;
      last.scale = (inverse && (pl->flags & EFFT_FLAG_SCALE_INVERSE)) ? 1.0 / (double)pl->col_len : 1.0;
      (void)inverse;
    }
    ns *= radices[p];
    CUDA_TRY(cudaFuncSetAttribute(pp.k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pp.k.smem_bytes));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pp.k.fn, pp.k.nt, pp.k.smem_bytes));
    if (occ < 1) return fail(EFFT_ERR_CUDA, "kernel does not fit on an SM (smem %d)", pp.k.smem_bytes);
    int64_t grid = (int64_t)occ * pl->num_sms;
    if (grid > pp.args.total_tasks) grid = pp.args.total_tasks;
    pp.grid = (int)grid;
    PassArgs& a = pp.args;
    if (pp.staged) {
      // Tasks are grabbed in order; ~grid of them are in flight at once.  B(g)
      // is issued `lag` steps after A(g) so its producers are done, and A(g)
      // reuses the slot of group g - slots, issued slots - lag steps earlier,
      // so slots - lag must also exceed the in-flight window.
      const int64_t per = a.a.ntasks + a.b.ntasks;
      const int64_t inflight = grid * 3;  // a warp-specialised CTA holds up to 3 tasks
      const int64_t window = (inflight + per - 1) / per;
      int64_t lag = env_int("EFFT_LAG", (int)(window + 1));
      if (lag < 1) lag = 1;
      if (lag > a.ngroups) lag = a.ngroups;
      int64_t slots = env_int("EFFT_SLOTS", (int)(lag + window + 2));
      if (slots < lag + 1) slots = lag + 1;
      if (slots > a.ngroups) slots = a.ngroups;
      a.lag = (int32_t)lag;
      a.nowait = env_int("EFFT_DIAG_NOWAIT", 0);  // diagnostics: 1 skip waits, 2 skip DFT work
      a.nslots = (int32_t)slots;
      size_t sb = (size_t)slots * a.slot_elems * pl->elem;
      if (sb > staging_bytes) staging_bytes = sb;
      pp.counter_off = coff;
      pp.counter_len = 2 + 2 * a.ngroups;
    } else {
      pp.counter_off = coff;
      pp.counter_len = 2;
    }
    coff += pp.counter_len;
  }
  pl->staging_bytes = staging_bytes;
  pl->counter_bytes = (size_t)coff * 4;
  return EFFT_OK;
}

}  // namespace

int finish_plan(efft_plan_s* pl) {
  int rc = EFFT_OK;
  if (rc == EFFT_OK && pl->staging_bytes) {
    if (cudaMalloc(&pl->staging, pl->staging_bytes) != cudaSuccess) {
      cudaGetLastError();
      rc = fail(EFFT_ERR_ALLOC, "staging ring of %zu bytes", pl->staging_bytes);
    }
  }
  if (rc == EFFT_OK && cudaMalloc((void**)&pl->counters, pl->counter_bytes) != cudaSuccess) {
    cudaGetLastError();
    rc = fail(EFFT_ERR_ALLOC, "counters");
  }
  if (rc == EFFT_OK && cudaMalloc((void**)&pl->flag, 4) != cudaSuccess) {
    cudaGetLastError();
    rc = fail(EFFT_ERR_ALLOC, "flag");
  }
  if (rc == EFFT_OK && cudaMemset(pl->flag, 0, 4) != cudaSuccess) rc = fail(EFFT_ERR_CUDA, "memset flag");
  if (rc != EFFT_OK) {
    std::string keep = g_err;
    efft_plan_destroy(pl);
    g_err = keep;
    return rc;
  }
  if (pl->tp) {
    int64_t off = 0;
    for (auto& q : pl->tpp) {
      q.a.stg = pl->staging;
      q.a.ctr = reinterpret_cast<unsigned long long*>(pl->counters + off);
      q.a.doneA = pl->counters + off + 2;
      q.a.doneB = q.a.doneA + q.a.ngroups;
      q.a.flag = pl->flag;
      off += q.counter_ints;
    }
    if (efft::tpass::encode_ring(pl->tpp[0], pl->staging) != 0) {
      efft_plan_destroy(pl);
      return fail(EFFT_ERR_CUDA, "tensor map (TMA pass ring) encode failed");
    }
    return EFFT_OK;
  }
  if (pl->lean) {
    int64_t off = 0;
    for (int i = 0; i < 2; ++i) {
      auto& q = pl->lp[i];
      q.a.stg = pl->staging;
      q.a.ctr = reinterpret_cast<unsigned long long*>(pl->counters + off);
      q.a.doneA = pl->counters + off + 2;
      q.a.doneB = q.a.doneA + q.a.ngroups;
      q.a.flag = pl->flag;
      off += q.counter_ints;
      if (q.pf && i == 0 && efft::lean::encode_ring(q, pl->staging) != 0) {
        efft_plan_destroy(pl);
        return fail(EFFT_ERR_CUDA, "tensor map (lean prefetch ring) encode failed");
      }
    }
    return EFFT_OK;
  }
  for (int p = 0; p < pl->npass; ++p) {
    PassArgs& a = pl->pass[p].args;
    a.staging = pl->staging;
    if (pl->pass[p].staged && pl->pass[p].k.ws) {
      int r2 = encode_B(pl, pl->pass[p]);
      if (r2 != EFFT_OK) {
        std::string keep = g_err;
        efft_plan_destroy(pl);
        g_err = keep;
        return r2;
      }
    }
    a.task_counter = reinterpret_cast<unsigned long long*>(pl->counters + pl->pass[p].counter_off);
    a.doneA = pl->counters + pl->pass[p].counter_off + 2;
    a.doneB = a.doneA + a.ngroups;
    a.flag = pl->flag;
  }
  return EFFT_OK;
}

extern "C" {

int efft_version(void) { return 1; }

const char* efft_last_error(void) { return g_err.c_str(); }

int efft_plan_create(efft_plan_t* out, int64_t n, int dtype, int direction, int device,
                     uint32_t flags) {
  if (!out) return fail(EFFT_ERR_INVALID_ARG, "plan pointer is NULL");
  *out = nullptr;
  if (dtype != EFFT_C64 && dtype != EFFT_C128 && dtype != EFFT_R32)
    return fail(EFFT_ERR_INVALID_ARG, "dtype %d", dtype);
  if (dtype == EFFT_R32 && direction != EFFT_FORWARD)
    return fail(EFFT_ERR_INVALID_ARG, "the real-input path is forward only");
  if (dtype == EFFT_R32 && (n < 4 || (n & 1)))
    return fail(EFFT_ERR_UNSUPPORTED_SIZE, "real-input n must be even and >= 4, got %lld", (long long)n);
  if (direction != EFFT_FORWARD && direction != EFFT_INVERSE)
    return fail(EFFT_ERR_INVALID_ARG, "direction must be -1 or +1, got %d", direction);
  if (n < 1) return fail(EFFT_ERR_INVALID_ARG, "n must be >= 1");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(EFFT_ERR_INVALID_ARG, "device %d of %d", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  efft_plan_s* pl = new efft_plan_s();
  pl->n_user = n;
  pl->real_input = dtype == EFFT_R32;
  pl->n = pl->real_input ? n / 2 : n;
  if (pl->real_input) dtype = EFFT_C64;
  pl->dtype = dtype;
  pl->direction = direction;
  pl->device = device;
  pl->flags = flags;
  pl->elem = dtype == EFFT_C64 ? 8 : 16;
  cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, device);
  int rc = build_plan(pl);
  if (rc != EFFT_OK) {
    delete pl;
    return rc;
  }
  rc = finish_plan(pl);  // frees the plan itself on failure
  if (rc != EFFT_OK) return rc;
  *out = pl;
  return EFFT_OK;
}

int efft_plan_create_columns(efft_plan_t* out, int64_t len, int64_t cols, int dtype, int direction, int device,
                             int64_t tw_mod, int64_t tw_offset, uint32_t flags) {
  if (!out) return fail(EFFT_ERR_INVALID_ARG, "plan pointer is NULL");
  *out = nullptr;
  if (dtype != EFFT_C64 && dtype != EFFT_C128) return fail(EFFT_ERR_INVALID_ARG, "dtype %d", dtype);
  if (direction != EFFT_FORWARD && direction != EFFT_INVERSE)
    return fail(EFFT_ERR_INVALID_ARG, "direction must be -1 or +1, got %d", direction);
  if (len < 2 || cols < 2) return fail(EFFT_ERR_INVALID_ARG, "len and cols must be >= 2");
  if (tw_mod < 0 || tw_offset < 0) return fail(EFFT_ERR_INVALID_ARG, "negative twiddle parameters");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(EFFT_ERR_INVALID_ARG, "device %d of %d", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  efft_plan_s* pl = new efft_plan_s();
  pl->columns = true;
  pl->col_len = len;
  pl->col_count = cols;
  pl->col_tw_mod = tw_mod;
  pl->col_tw_offset = tw_offset;
  pl->n = pl->n_user = len * cols;
  pl->dtype = dtype;
  pl->direction = direction;
  pl->device = device;
  pl->flags = flags;
  pl->elem = dtype == EFFT_C64 ? 8 : 16;
  cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, device);
  int rc = build_plan(pl);
  if (rc != EFFT_OK) {
    delete pl;
    return rc;
  }
  rc = finish_plan(pl);  // frees the plan itself on failure
  if (rc != EFFT_OK) return rc;
  *out = pl;
  return EFFT_OK;
}

int efft_permute_swap01(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, int elem_bytes,
                        void* stream) {
  if (!in || !out || in == out) return fail(EFFT_ERR_INVALID_ARG, "bad buffers");
  if (n0 < 1 || n1 < 1 || n2 < 1 || (elem_bytes != 8 && elem_bytes != 16))
    return fail(EFFT_ERR_INVALID_ARG, "bad shape");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t words = n0 * n1 * n2 * elem_bytes / 16;
  const unsigned grid = (unsigned)std::min<int64_t>((words + 255) / 256, 148 * 32);
  if ((n2 * elem_bytes) % 16 == 0)
    efft::swap01_kernel<uint4><<<grid, 256, 0, s>>>((const uint4*)in, (uint4*)out, n0, n1, n2 * elem_bytes / 16);
  else
    efft::swap01_kernel<uint2><<<grid, 256, 0, s>>>((const uint2*)in, (uint2*)out, n0, n1, n2);
  CUDA_TRY(cudaGetLastError());
  return EFFT_OK;
}

int efft_permute_swap12(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, int elem_bytes,
                        void* stream) {
  if (!in || !out || in == out) return fail(EFFT_ERR_INVALID_ARG, "bad buffers");
  if (n0 < 1 || n1 < 1 || n2 < 1 || (elem_bytes != 8 && elem_bytes != 16) || n0 > 65535)
    return fail(EFFT_ERR_INVALID_ARG, "bad shape");
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)((n2 + 31) / 32), (unsigned)((n1 + 31) / 32), (unsigned)n0), block(32, 8);
  if (elem_bytes == 16)
    efft::swap12_kernel<uint4><<<grid, block, 0, s>>>((const uint4*)in, (uint4*)out, n1, n2);
  else
    efft::swap12_kernel<uint2><<<grid, block, 0, s>>>((const uint2*)in, (uint2*)out, n1, n2);
  CUDA_TRY(cudaGetLastError());
  return EFFT_OK;
}

int efft_plan_describe(efft_plan_t pl, char* buf, size_t len) {
  if (!pl || !buf) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  std::string s;
  char line[512];
  snprintf(line, sizeof line, "n=%lld dtype=%s direction=%d passes=%d staging=%zu B\n",
           (long long)pl->n, pl->dtype == EFFT_C64 ? "c64" : "c128", pl->direction, pl->npass,
           pl->staging_bytes);
  s += line;
  for (int p = 0; pl->tp && p < 2; ++p) {
    const efft::tpass::Pass& q = pl->tpp[p];
    snprintf(line, sizeof line,
             "pass %d: R=%lld tma staged rho_a=256 rho_b=%d stages=[16x16 | 8x16] F=32 grid=%d x %d smem=%d "
             "groups=%d tasks=%lld lag=%d slots=%d\n",
             p, (long long)q.a.R, q.rb, q.grid, q.nt, q.smem, q.a.ngroups, (long long)q.a.total, q.a.lag,
             q.a.nslots);
    s += line;
  }
  for (int p = 0; pl->lean && p < 2; ++p) {
    const efft::lean::Pass& q = pl->lp[p];
    snprintf(line, sizeof line,
             "pass %d: R=%lld lean staged rho_a=%d rho_b=%d stages=[%dx%d | %dx16] grid=%d x %d smem=%d "
             "groups=%d tasks=%lld lag=%d slots=%d\n",
             p, (long long)q.a.R, q.ra, q.rb, q.ra / 16, 16, q.rb / 16, q.grid, q.nt, q.smem, q.a.ngroups,
             (long long)q.a.total,
             q.a.lag, q.a.nslots);
    s += line;
  }
  for (int p = 0; !pl->lean && !pl->tp && p < pl->npass; ++p) {
    const PassPlan& pp = pl->pass[p];
    std::string st;
    for (int i = 0; i < pp.k.nst_a; ++i) st += (i ? "x" : "") + std::to_string(pp.k.stages_a[i]);
    if (pp.staged) {
      st += " | ";
      for (int i = 0; i < pp.k.nst_b; ++i) st += (i ? "x" : "") + std::to_string(pp.k.stages_b[i]);
    }
    snprintf(line, sizeof line,
             "pass %d: R=%lld %s rho_a=%lld rho_b=%lld stages=[%s] grid=%d x %d smem=%d groups=%lld "
             "tasks=%lld lag=%d slots=%d\n",
             p, (long long)pp.radix, pp.staged ? "staged" : "direct", (long long)pp.rho_a,
             (long long)pp.rho_b, st.c_str(), pp.grid, pp.k.nt, pp.k.smem_bytes,
             (long long)pp.args.ngroups, (long long)pp.args.total_tasks, pp.args.lag, pp.args.nslots);
    s += line;
  }
  snprintf(buf, len, "%s", s.c_str());
  return EFFT_OK;
}

int efft_plan_workspace_bytes(efft_plan_t pl, size_t* bytes) {
  if (!pl || !bytes) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  *bytes = pl->staging_bytes + pl->counter_bytes + 4;
  for (const auto& r : pl->ranks)  // sharded: per rank, work array + ring + counters
    *bytes += (size_t)(pl->n / (int64_t)pl->ranks.size()) * pl->elem +
              (size_t)std::max(r.lp[0].a.nslots * r.lp[0].a.slot_elems, r.lp[1].a.nslots * r.lp[1].a.slot_elems) *
                  pl->elem +
              r.counter_bytes + 4;
  return EFFT_OK;
}

int efft_plan_launches(efft_plan_t pl, int* launches) {
  if (!pl || !launches) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  *launches = pl->npass + (pl->real_input ? 1 : 0);
  return EFFT_OK;
}

int efft_execute(efft_plan_t pl, const void* d_in, void* d_out, void* stream) {
  if (!pl || !d_in || !d_out) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  const size_t bytes = (size_t)pl->n * pl->elem;
  const char* i0 = (const char*)d_in;
  const char* o0 = (const char*)d_out;
  // column plans are one position-preserving pass: in place is allowed
  if (!(pl->columns && d_in == d_out) && i0 < o0 + bytes && o0 < i0 + bytes)
    return fail(EFFT_ERR_INVALID_ARG, "input and output overlap");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(pl->device));
  CUDA_TRY(cudaMemsetAsync(pl->counters, 0, pl->counter_bytes, s));
  cudaEvent_t* ev = pl->timing ? &pl->tev[(size_t)(pl->tcount % pl->tcap) * 4] : nullptr;
  if (pl->timing) ++pl->tcount;
  for (int p = 0; pl->tp && p < 2; ++p) {
    if (ev) CUDA_TRY(cudaEventRecord(ev[p], s));
    efft::tpass::Pass& q = pl->tpp[p];
    const void* src = p == 0 ? d_in : d_out;
    if (q.mapA_ptr != src && efft::tpass::encode_input(q, p, src) != 0)
      return fail(EFFT_ERR_CUDA, "tensor map (TMA pass input) encode failed");
    efft::tpass::Args a = q.a;
    a.src = src;
    a.dst = d_out;
    static const bool tprof = getenv("EFFT_TP_PROF") != nullptr;
    if (tprof) {  // diagnostics: per-phase cycle sums of this launch, printed to stderr
      static unsigned long long* buf = nullptr;
      if (!buf) CUDA_TRY(cudaMalloc(&buf, 96 * 8));
      CUDA_TRY(cudaMemsetAsync(buf, 0, 96 * 8, s));
      a.prof = buf;
      q.fn_prof<<<q.grid, q.nt, q.smem, s>>>(a);
      CUDA_TRY(cudaGetLastError());
      unsigned long long h[96];
      CUDA_TRY(cudaMemcpyAsync(h, buf, sizeof h, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      const double ctas = q.grid;
      fprintf(stderr,
              "tpass pass %d (per CTA): producer dep-wait %.0f, buffer-wait %.0f, total %.0f cycles; "
              "deferred %.1f of %.1f tiles; compute warp 0: tile-wait %.0f, barrier %.0f, total %.0f\n",
              p, h[0] / ctas, h[1] / ctas, h[2] / ctas, h[6] / ctas, h[7] / ctas, h[3] / ctas, h[4] / ctas,
              (double)h[5] / ctas);
      for (int k = 0; k < 2; ++k) {
        fprintf(stderr, "  compute warp 0 %s tiles, cycles per tile [ld, st0, bar+sts+bar, ld1, st1+stores, end]:",
                k ? "B" : "A");
        for (int i = 0; i < 6; ++i) fprintf(stderr, " %.0f", h[8 + k * 6 + i] / ctas / (h[7] / ctas / 2));
        fprintf(stderr, "\n");
      }
      continue;
    }
    q.fn<<<q.grid, q.nt, q.smem, s>>>(a);
    CUDA_TRY(cudaGetLastError());
  }
  for (int p = 0; pl->lean && p < 2; ++p) {
    if (ev) CUDA_TRY(cudaEventRecord(ev[p], s));
    efft::lean::Pass& q = pl->lp[p];
    const void* src = p == 0 ? d_in : d_out;
    if (q.pf && q.mapA_ptr != src && efft::lean::encode_input(q, src) != 0)
      return fail(EFFT_ERR_CUDA, "tensor map (lean prefetch input) encode failed");
    efft::lean::Args a = q.a;
    a.src = src;
    a.dst = d_out;
    q.fn<<<q.grid, q.nt, q.smem, s>>>(a);
    CUDA_TRY(cudaGetLastError());
  }
  for (int p = 0; !pl->lean && !pl->tp && p < pl->npass; ++p) {
    if (ev) CUDA_TRY(cudaEventRecord(ev[p], s));
    PassPlan& pp = pl->pass[p];
    const void* src = p == 0 ? d_in : d_out;
    if (pp.k.ws && pp.tmA_ptr != src) {
      int rc = pp.staged ? encode_A(pl, pp, src) : encode_D(pl, pp, src);
      if (rc != EFFT_OK) return rc;
    }
    PassArgs a = pp.args;
    a.in = src;
    a.out = d_out;
    pp.k.fn<<<pp.grid, pp.k.nt, pp.k.smem_bytes, s>>>(a);
    CUDA_TRY(cudaGetLastError());
  }
  if (ev) CUDA_TRY(cudaEventRecord(ev[pl->npass], s));
  if (pl->real_input) {
    const int64_t h = pl->n, pairs = h / 2 + 1;
    const int64_t threads = (pairs + SPLIT_K - 1) / SPLIT_K;
    real_split_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>((float2*)d_out, h, pl->n_user);
    CUDA_TRY(cudaGetLastError());
    if (ev) CUDA_TRY(cudaEventRecord(ev[pl->npass + 1], s));
  }
  return EFFT_OK;
}

int efft_execute_host(efft_plan_t pl, const void* h_in, void* h_out, void* stream) {
  if (!pl || !h_in || !h_out) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  CUDA_TRY(cudaSetDevice(pl->device));
  const size_t bytes = (size_t)pl->n * pl->elem;
  // The device in/out pair is shared by every plan of the device (one pool,
  // grown on demand), so a forward and an inverse plan of a 64 GiB transform
  // need 128 GiB between them, not 256.  The call is synchronous and holds the
  // pool's lock until its copies are done.
  HostPool& hp = host_pool(pl->device);
  std::lock_guard<std::mutex> lock(hp.mu);
  if (hp.bytes < bytes) {
    if (hp.in) cudaFree(hp.in);
    if (hp.out) cudaFree(hp.out);
    hp.in = hp.out = nullptr;
    hp.bytes = 0;
    if (cudaMalloc(&hp.in, bytes) != cudaSuccess || cudaMalloc(&hp.out, bytes) != cudaSuccess) {
      cudaGetLastError();
      if (hp.in) cudaFree(hp.in);
      hp.in = nullptr;
      return fail(EFFT_ERR_ALLOC, "device buffers for host execution (%zu bytes each)", bytes);
    }
    hp.bytes = bytes;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(hp.in, h_in, bytes, cudaMemcpyHostToDevice, s));
  int rc = efft_execute(pl, hp.in, hp.out, stream);
  if (rc != EFFT_OK) return rc;
  CUDA_TRY(cudaMemcpyAsync(h_out, hp.out, bytes, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return EFFT_OK;
}

int efft_execute_host_batch(efft_plan_t pl, const void* const* h_in, void* const* h_out, int count, void* stream) {
  if (!pl || !h_in || !h_out || count < 1) return fail(EFFT_ERR_INVALID_ARG, "NULL argument or count < 1");
  for (int k = 0; k < count; ++k)
    if (!h_in[k] || !h_out[k]) return fail(EFFT_ERR_INVALID_ARG, "NULL host buffer %d", k);
  CUDA_TRY(cudaSetDevice(pl->device));
  const size_t bytes = (size_t)pl->n * pl->elem;
  if (count == 1) return efft_execute_host(pl, h_in[0], h_out[0], stream);
  HostPool& hp = host_pool(pl->device);
  std::lock_guard<std::mutex> lock(hp.mu);
  // two device in/out pairs from the per-device pool (grown on demand; when
  // they do not fit, one transform at a time through the first pair)
  auto grow = [&](void*& i, void*& o, size_t& have) -> bool {
    if (have >= bytes) return true;
    if (i) cudaFree(i);
    if (o) cudaFree(o);
    i = o = nullptr;
    have = 0;
    if (cudaMalloc(&i, bytes) != cudaSuccess || cudaMalloc(&o, bytes) != cudaSuccess) {
      cudaGetLastError();
      if (i) cudaFree(i);
      i = nullptr;
      return false;
    }
    have = bytes;
    return true;
  };
  if (!grow(hp.in, hp.out, hp.bytes)) return fail(EFFT_ERR_ALLOC, "device buffers for host execution (%zu bytes each)", bytes);
  cudaStream_t s = (cudaStream_t)stream;
  if (!grow(hp.in2, hp.out2, hp.bytes2)) {  // sequential fallback
    for (int k = 0; k < count; ++k) {
      CUDA_TRY(cudaMemcpyAsync(hp.in, h_in[k], bytes, cudaMemcpyHostToDevice, s));
      int rc = efft_execute(pl, hp.in, hp.out, stream);
      if (rc != EFFT_OK) return rc;
      CUDA_TRY(cudaMemcpyAsync(h_out[k], hp.out, bytes, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    return EFFT_OK;
  }
  if (!hp.cs) CUDA_TRY(cudaStreamCreateWithFlags(&hp.cs, cudaStreamNonBlocking));
  for (auto& e : hp.ev)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // Transform k+1's H2D (copy stream) overlaps transform k's passes and D2H
  // (the caller's stream): the two PCIe directions run concurrently.
  void* din[2] = {hp.in, hp.in2};
  void* dout[2] = {hp.out, hp.out2};
  cudaEvent_t in_ready[2] = {hp.ev[0], hp.ev[1]}, buf_free[2] = {hp.ev[2], hp.ev[3]};
  CUDA_TRY(cudaEventRecord(buf_free[0], s));
  CUDA_TRY(cudaEventRecord(buf_free[1], s));
  for (int k = 0; k < count; ++k) {
    const int b = k & 1;
    CUDA_TRY(cudaStreamWaitEvent(hp.cs, buf_free[b], 0));
    CUDA_TRY(cudaMemcpyAsync(din[b], h_in[k], bytes, cudaMemcpyHostToDevice, hp.cs));
    CUDA_TRY(cudaEventRecord(in_ready[b], hp.cs));
    CUDA_TRY(cudaStreamWaitEvent(s, in_ready[b], 0));
    int rc = efft_execute(pl, din[b], dout[b], stream);
    if (rc != EFFT_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(h_out[k], dout[b], bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(buf_free[b], s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  return EFFT_OK;
}

// ---- out-of-core transform ----------------------------
// N = N1 N2 (N1 takes the odd factor), x viewed as (N1 x N2) row-major.
//   step 1  per block of C columns n2: strided H2D DMA of x[:, c0:c0+C], a
//           column plan of length N1, a device transpose -> rows c0.. of
//           Yt[n2][k1] (= h_out, contiguous D2H)
//   step 2  per block of Rr columns k1 of Yt: strided H2D DMA, a column plan
//           of length N2 with the four-step twiddle W_N^(n2 k1), strided D2H
//           into the SAME columns of h_out viewed as X[k2][k1]
// Step 2 reads each block of h_out exactly where it writes it back, so the
// host intermediate costs no memory.  Blocks alternate between two streams and
// two device buffer sets: one block's H2D overlaps the other's D2H and plan.
// The host buffers are page-locked for the call (cudaHostRegister) so every
// copy is a DMA straight from / to the caller's arrays.
namespace {
int64_t ooc_fit(int64_t length, int64_t dim, int64_t per, int64_t f) {
  int64_t b = std::max(f, std::min(dim, per / length));
  b -= b % f;
  b = std::max(f, b);
  while (b >= f && dim % b) b -= f;
  return (b >= f && dim % b == 0) ? b : 0;
}
}  // namespace

int efft_outofcore_blocks(int64_t n, int dtype, size_t device_bytes, int64_t* blocks) {
  if (!blocks) return fail(EFFT_ERR_INVALID_ARG, "blocks is NULL");
  if (dtype != EFFT_C64 && dtype != EFFT_C128) return fail(EFFT_ERR_INVALID_ARG, "dtype %d", dtype);
  int M, t;
  if (n < 4 || !factor(n, &M, &t)) return fail(EFFT_ERR_UNSUPPORTED_SIZE, "n=%lld is not M*2^t with M in {1,3,5,7}", (long long)n);
  const int t1 = t / 2;
  const int64_t n1 = (int64_t)M << t1, n2 = (int64_t)1 << (t - t1);
  if (n1 > (1 << 17) || n2 > (1 << 17))
    return fail(EFFT_ERR_UNSUPPORTED_SIZE, "n=%lld exceeds the out-of-core range (N1, N2 <= 2^17)", (long long)n);
  const int64_t e = dtype == EFFT_C64 ? 8 : 16, f = dtype == EFFT_C64 ? 16 : 8;
  const int64_t per = std::max<int64_t>(1, (int64_t)(device_bytes / (4 * e)));  // 2 streams x 2 buffers
  const int64_t cb = ooc_fit(n1, n2, per, f), rb = ooc_fit(n2, n1, per, f);
  if (!cb || !rb) return fail(EFFT_ERR_UNSUPPORTED_SIZE, "no block of n=%lld fits %zu bytes", (long long)n, device_bytes);
  blocks[0] = n1;
  blocks[1] = n2;
  blocks[2] = cb;
  blocks[3] = rb;
  return EFFT_OK;
}

int efft_execute_outofcore(int64_t n, int dtype, int direction, int device, uint32_t flags, const void* h_in,
                           void* h_out, size_t device_bytes) {
  if (!h_in || !h_out) return fail(EFFT_ERR_INVALID_ARG, "NULL host buffer");
  if (direction != EFFT_FORWARD && direction != EFFT_INVERSE)
    return fail(EFFT_ERR_INVALID_ARG, "direction must be -1 or +1, got %d", direction);
  int64_t bl[4];
  int rc = efft_outofcore_blocks(n, dtype, device_bytes, bl);
  if (rc != EFFT_OK) return rc;
  const int64_t n1 = bl[0], n2 = bl[1], cb = bl[2], rb = bl[3];
  const size_t e = dtype == EFFT_C64 ? 8 : 16, bytes = (size_t)n * e;
  const char* hi = (const char*)h_in;
  char* ho = (char*)h_out;
  if (hi < ho + bytes && ho < hi + bytes) return fail(EFFT_ERR_INVALID_ARG, "input and output overlap");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(EFFT_ERR_INVALID_ARG, "device %d of %d", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  struct Res {  // released on every exit path
    efft_plan_t p1[2] = {nullptr, nullptr}, p2[2] = {nullptr, nullptr};
    void* a[2] = {nullptr, nullptr};
    void* b[2] = {nullptr, nullptr};
    cudaStream_t s[2] = {nullptr, nullptr};
    void* reg[2] = {nullptr, nullptr};
    void* stage[2] = {nullptr, nullptr};  // pinned step-1 staging when h_in cannot be page-locked
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Res() {
      for (int i = 0; i < 2; ++i) {
        if (s[i]) cudaStreamSynchronize(s[i]);
      }
      for (int i = 0; i < 2; ++i) {
        if (p1[i]) efft_plan_destroy(p1[i]);
        if (p2[i]) efft_plan_destroy(p2[i]);
        if (a[i]) cudaFree(a[i]);
        if (b[i]) cudaFree(b[i]);
        if (s[i]) cudaStreamDestroy(s[i]);
        if (reg[i]) cudaHostUnregister(reg[i]);
        if (stage[i]) cudaFreeHost(stage[i]);
        if (ev[i]) cudaEventDestroy(ev[i]);
      }
    }
  } r;
  bool staged_in = false;
  for (int i = 0; i < 2; ++i) {
    void* ptr = i == 0 ? (void*)hi : (void*)ho;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost) continue;  // caller-pinned
    cudaGetLastError();
    cudaError_t er = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (er != cudaSuccess && er != cudaErrorHostMemoryAlreadyRegistered && i == 0) {
      // read-only pages (e.g. a read-only mapping of the input file): step 1
      // gathers its blocks through pinned staging buffers instead
      cudaGetLastError();
      staged_in = true;
      continue;
    }
    if (er == cudaSuccess) r.reg[i] = ptr;
    else if (er == cudaErrorHostMemoryAlreadyRegistered) cudaGetLastError();  // caller-pinned: keep as is
    else {
      cudaGetLastError();
      return fail(EFFT_ERR_CUDA, "cudaHostRegister of %zu bytes: %s", bytes, cudaGetErrorString(er));
    }
  }
  const size_t buf = (size_t)std::max(n1 * cb, n2 * rb) * e;
  const uint32_t pf = flags & (EFFT_FLAG_SCALE_INVERSE | EFFT_FLAG_CHECK_FINITE);
  for (int i = 0; i < 2; ++i) {
    if (cudaMalloc(&r.a[i], buf) != cudaSuccess || cudaMalloc(&r.b[i], buf) != cudaSuccess) {
      cudaGetLastError();
      return fail(EFFT_ERR_ALLOC, "out-of-core device buffers (4 x %zu bytes)", buf);
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&r.s[i], cudaStreamNonBlocking));
    if (staged_in) {
      if (cudaHostAlloc(&r.stage[i], (size_t)(n1 * cb) * e, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return fail(EFFT_ERR_ALLOC, "out-of-core pinned staging (2 x %zu bytes)", (size_t)(n1 * cb) * e);
      }
      CUDA_TRY(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming));
    }
    rc = efft_plan_create_columns(&r.p1[i], n1, cb, dtype, direction, device, 0, 0, pf);
    if (rc != EFFT_OK) return rc;
    rc = efft_plan_create_columns(&r.p2[i], n2, rb, dtype, direction, device, n, 0, pf);
    if (rc != EFFT_OK) return rc;
  }
  // step 1
  for (int64_t c0 = 0, k = 0; c0 < n2; c0 += cb, ++k) {
    const int i = (int)(k & 1);
    if (staged_in) {  // host gather of block k overlaps the device work of block k-1
      if (k >= 2) CUDA_TRY(cudaEventSynchronize(r.ev[i]));
      char* st = (char*)r.stage[i];
      for (int64_t row = 0; row < n1; ++row) memcpy(st + row * cb * e, hi + (row * n2 + c0) * e, cb * e);
      CUDA_TRY(cudaMemcpyAsync(r.a[i], st, (size_t)(n1 * cb) * e, cudaMemcpyHostToDevice, r.s[i]));
      CUDA_TRY(cudaEventRecord(r.ev[i], r.s[i]));
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(r.a[i], cb * e, hi + c0 * e, n2 * e, cb * e, n1, cudaMemcpyHostToDevice, r.s[i]));
    }
    rc = efft_execute(r.p1[i], r.a[i], r.a[i], r.s[i]);
    if (rc != EFFT_OK) return rc;
    rc = efft_permute_swap01(r.a[i], r.b[i], n1, cb, 1, (int)e, r.s[i]);  // [k1][c] -> [c][k1]
    if (rc != EFFT_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(ho + c0 * n1 * e, r.b[i], cb * n1 * e, cudaMemcpyDeviceToHost, r.s[i]));
  }
  for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamSynchronize(r.s[i]));
  if (pf & EFFT_FLAG_CHECK_FINITE) {  // the reference rejects non-finite input (scatter.py:38-39)
    for (int i = 0; i < 2; ++i) {
      int seen = 0;
      rc = efft_nonfinite_seen(r.p1[i], &seen, r.s[i]);
      if (rc != EFFT_OK) return rc;
      if (seen) return fail(EFFT_ERR_INVALID_ARG, "input contains non-finite values");
    }
  }
  // step 2 (the twiddle offset of a column plan is the first k1 of its block)
  for (int64_t r0 = 0, k = 0; r0 < n1; r0 += rb, ++k) {
    const int i = (int)(k & 1);
    efft_plan_s* p2 = r.p2[i];
    p2->col_tw_offset = r0;
    p2->pass[0].args.a.A0 = r0;
    CUDA_TRY(cudaMemcpy2DAsync(r.a[i], rb * e, ho + r0 * e, n1 * e, rb * e, n2, cudaMemcpyHostToDevice, r.s[i]));
    rc = efft_execute(p2, r.a[i], r.a[i], r.s[i]);
    if (rc != EFFT_OK) return rc;
    CUDA_TRY(cudaMemcpy2DAsync(ho + r0 * e, n1 * e, r.a[i], rb * e, rb * e, n2, cudaMemcpyDeviceToHost, r.s[i]));
  }
  for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamSynchronize(r.s[i]));
  return EFFT_OK;
}

int efft_release_host_buffers(int device) {
  if (device < 0 || device >= kMaxDevices) return fail(EFFT_ERR_INVALID_ARG, "device %d", device);
  HostPool& hp = host_pool(device);
  std::lock_guard<std::mutex> lock(hp.mu);
  CUDA_TRY(cudaSetDevice(device));
  if (hp.in) cudaFree(hp.in);
  if (hp.out) cudaFree(hp.out);
  if (hp.in2) cudaFree(hp.in2);
  if (hp.out2) cudaFree(hp.out2);
  hp.in = hp.out = hp.in2 = hp.out2 = nullptr;
  hp.bytes = hp.bytes2 = 0;
  return EFFT_OK;
}

int efft_nonfinite_seen(efft_plan_t pl, int* seen, void* stream) {
  if (!pl || !seen) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  CUDA_TRY(cudaSetDevice(pl->device));
  cudaStream_t s = (cudaStream_t)stream;
  int32_t v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, pl->flag, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaMemsetAsync(pl->flag, 0, 4, s));
  *seen = v != 0;
  return EFFT_OK;
}

int efft_plan_enable_timing(efft_plan_t pl, int enable) {
  if (!pl) return fail(EFFT_ERR_INVALID_ARG, "NULL plan");
  if (enable < 0) return fail(EFFT_ERR_INVALID_ARG, "enable must be >= 0, got %d", enable);
  CUDA_TRY(cudaSetDevice(pl->device));
  for (auto& e : pl->tev)
    if (e) cudaEventDestroy(e);
  pl->tev.clear();
  pl->tcap = enable;
  pl->tcount = 0;
  pl->timing = enable > 0;
  if (pl->timing) {
    pl->tev.assign((size_t)enable * 4, nullptr);
    for (auto& e : pl->tev) CUDA_TRY(cudaEventCreate(&e));
  }
  return EFFT_OK;
}

int efft_plan_launch_times(efft_plan_t pl, float* ms, int max_launches) {
  if (!pl || !ms) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  if (!pl->timing) return fail(EFFT_ERR_INVALID_ARG, "timing not enabled");
  if (pl->tcount == 0) return fail(EFFT_ERR_INVALID_ARG, "no timed execute yet");
  const int nl = pl->npass + (pl->real_input ? 1 : 0);
  const long long first = pl->tcount > pl->tcap ? pl->tcount - pl->tcap : 0;
  CUDA_TRY(cudaSetDevice(pl->device));
  for (int i = 0; i < nl && i < max_launches; ++i) {
    double sum = 0;
    for (long long j = first; j < pl->tcount; ++j) {
      const cudaEvent_t* ev = &pl->tev[(size_t)(j % pl->tcap) * 4];
      float t = 0;
      CUDA_TRY(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
      sum += t;
    }
    ms[i] = (float)(sum / (double)(pl->tcount - first));
  }
  return EFFT_OK;
}

static int launch_lean(efft::lean::Pass& q, const void* src, void* dst, cudaStream_t s, int64_t j2shift = 0) {
  efft::lean::Args a = q.a;
  a.src = src;
  a.dst = dst;
  a.j2off += j2shift;  // column chunk of the transposing pass: global column of its first column
  q.fn<<<q.grid, q.nt, q.smem, s>>>(a);
  CUDA_TRY(cudaGetLastError());
  return EFFT_OK;
}

int efft_plan_create_sharded(efft_plan_t* out, int64_t n, int dtype, int direction, int ngpus, const int* devices,
                             uint32_t flags) {
  if (!out) return fail(EFFT_ERR_INVALID_ARG, "plan pointer is NULL");
  *out = nullptr;
  if (dtype != EFFT_C64 && dtype != EFFT_C128) return fail(EFFT_ERR_INVALID_ARG, "dtype %d (complex only)", dtype);
  if (direction != EFFT_FORWARD && direction != EFFT_INVERSE)
    return fail(EFFT_ERR_INVALID_ARG, "direction must be -1 or +1, got %d", direction);
  if (ngpus < 1 || ngpus > 64 || (ngpus & (ngpus - 1)) || !devices)
    return fail(EFFT_ERR_INVALID_ARG, "ngpus must be a power of two in [1, 64] with a device list");
  const int c128 = dtype == EFFT_C128;
  int64_t N1, N2;
  if (!efft::lean::split_sharded(n, ngpus, c128, &N1, &N2))
    return fail(EFFT_ERR_UNSUPPORTED_SIZE, "n=%lld cannot be sharded over %d GPUs (N = N1 N2 with N1 = 2^a >= 2^12, "
                "N2 = M 2^b, G F | N1, N2)", (long long)n, ngpus);
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  for (int i = 0; i < ngpus; ++i)
    if (devices[i] < 0 || devices[i] >= ndev) return fail(EFFT_ERR_INVALID_ARG, "device %d of %d", devices[i], ndev);
  efft_plan_s* pl = new efft_plan_s();
  pl->n = pl->n_user = n;
  pl->dtype = dtype;
  pl->direction = direction;
  pl->device = devices[0];
  pl->flags = flags;
  pl->elem = c128 ? 16 : 8;
  pl->npass = 2;
  pl->sh_n1 = N1;
  pl->sh_n2 = N2;
  pl->ranks.resize(ngpus);
  const size_t local = (size_t)(n / ngpus) * pl->elem;
  // Column chunks of the overlapped schedule (EFFT_SHARD_CHUNKS, default 4): every
  // chunk keeps whole lane groups and at least 16 of them; 1 = the sequential schedule
  int chunks = env_int("EFFT_SHARD_CHUNKS", 4);
  {
    const int64_t L1 = N1 / ngpus, L2 = N2 / ngpus, F = efft::lean::lanes(c128);
    if (chunks < 1) chunks = 1;
    while (chunks > 1 && (L1 % (chunks * F) || L2 % (chunks * F) || L1 / (chunks * F) < 16 || L2 / (chunks * F) < 16))
      chunks /= 2;
  }
  pl->sh_chunks = chunks;
  for (int q = 0; q < ngpus; ++q) {
    auto& r = pl->ranks[q];
    r.dev = devices[q];
    if (cudaSetDevice(r.dev) != cudaSuccess) {
      efft_plan_destroy(pl);
      return fail(EFFT_ERR_CUDA, "cudaSetDevice(%d)", r.dev);
    }
    int sms = 0, ecuda = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, r.dev);
    int64_t stg = 0;
    if (!efft::lean::plan_sharded(n, ngpus, q, c128, direction == EFFT_INVERSE, (flags & EFFT_FLAG_CHECK_FINITE) != 0,
                                  sms, r.lp, &stg, &ecuda, false, chunks)) {
      efft_plan_destroy(pl);
      return ecuda ? fail(EFFT_ERR_CUDA, "sharded pass setup failed") : fail(EFFT_ERR_UNSUPPORTED_SIZE, "no pass kernel");
    }
    r.counter_bytes = (size_t)(r.lp[0].counter_ints + r.lp[1].counter_ints) * 4;
    if (cudaMalloc(&r.staging, (size_t)stg * pl->elem) != cudaSuccess ||
        cudaMalloc((void**)&r.counters, r.counter_bytes) != cudaSuccess || cudaMalloc((void**)&r.flag, 4) != cudaSuccess ||
        cudaMalloc(&r.work, local) != cudaSuccess || cudaMemset(r.flag, 0, 4) != cudaSuccess ||
        cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      efft_plan_destroy(pl);
      return fail(EFFT_ERR_ALLOC, "sharded rank %d buffers (%zu bytes + ring)", q, local);
    }
    if (chunks > 1) {
      bool ok = cudaMalloc(&r.work2, local) == cudaSuccess &&
                cudaStreamCreateWithFlags(&r.cs, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&r.cs2, cudaStreamNonBlocking) == cudaSuccess;
      r.cev.assign((size_t)5 * chunks, nullptr);
      for (auto& e : r.cev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
      if (!ok) {
        cudaGetLastError();
        efft_plan_destroy(pl);
        return fail(EFFT_ERR_ALLOC, "sharded rank %d overlap buffers (%zu bytes)", q, local);
      }
    }
    int64_t off = 0;
    for (auto& ps : r.lp) {
      ps.a.stg = r.staging;
      ps.a.ctr = reinterpret_cast<unsigned long long*>(r.counters + off);
      ps.a.doneA = r.counters + off + 2;
      ps.a.doneB = ps.a.doneA + ps.a.ngroups;
      ps.a.flag = r.flag;
      off += ps.counter_ints;
    }
    // peer access to every other device (the exchanges are pitched peer copies)
    for (int p = 0; p < ngpus; ++p) {
      if (devices[p] == r.dev) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, r.dev, devices[p]);
      if (can) {
        cudaError_t e = cudaDeviceEnablePeerAccess(devices[p], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          efft_plan_destroy(pl);
          return fail(EFFT_ERR_CUDA, "peer access %d -> %d: %s", r.dev, devices[p], cudaGetErrorString(e));
        }
        cudaGetLastError();
      }
    }
  }
  *out = pl;
  return EFFT_OK;
}

int efft_execute_sharded(efft_plan_t pl, const void* const* in, void* const* out, void* const* streams) {
  if (!pl || !in || !out || !streams) return fail(EFFT_ERR_INVALID_ARG, "NULL argument");
  if (pl->ranks.empty()) return fail(EFFT_ERR_INVALID_ARG, "not a sharded plan");
  const int G = (int)pl->ranks.size();
  const int64_t N1 = pl->sh_n1, N2 = pl->sh_n2, L1 = N1 / G, L2 = N2 / G;
  const size_t e = pl->elem;
  for (int q = 0; q < G; ++q)
    if (!in[q] || !out[q] || in[q] == out[q]) return fail(EFFT_ERR_INVALID_ARG, "rank %d: bad buffers", q);
  auto S = [&](int q) { return (cudaStream_t)streams[q]; };
  auto W = [&](int q) { return (char*)pl->ranks[q].work; };
  // every rank's stream waits for every rank's previous step (cross-device events)
  auto all_wait = [&]() -> int {
    for (int q = 0; q < G; ++q) {
      CUDA_TRY(cudaSetDevice(pl->ranks[q].dev));
      CUDA_TRY(cudaEventRecord(pl->ranks[q].ev, S(q)));
    }
    for (int q = 0; q < G; ++q) {
      CUDA_TRY(cudaSetDevice(pl->ranks[q].dev));
      for (int p = 0; p < G; ++p)
        if (p != q) CUDA_TRY(cudaStreamWaitEvent(S(q), pl->ranks[p].ev, 0));
    }
    return EFFT_OK;
  };
  int rc = all_wait();
  if (rc != EFFT_OK) return rc;
  if (pl->sh_chunks > 1) {
    // Overlapped schedule: the local passes run in C column chunks on the caller's
    // streams while the exchanges of the neighbouring chunks run on per-rank copy
    // streams (pitched peer copies over NVLink):
    //   exchange 1 chunk i+1  ||  pass 1 chunk i  ||  exchange 2 slab i-1
    //   pass 2 chunk j        ||  exchange 3 slab j-1
    // Exchange 2 lands in a second work array (pass 1 of the destination may still be
    // reading its first one).  Exposed: the first chunk of exchange 1, the last slab of
    // exchange 2 (pass 2 needs every row) and the last slab of exchange 3.
    const int C = pl->sh_chunks;
    const int64_t c2 = L2 / C, c1 = L1 / C;
    auto CS = [&](int q) { return pl->ranks[q].cs; };
    auto CO = [&](int q) { return pl->ranks[q].cs2; };
    auto W2 = [&](int q) { return (char*)pl->ranks[q].work2; };
    auto EV = [&](int q, int kind, int i) { return pl->ranks[q].cev[(size_t)kind * C + i]; };
    for (int q = 0; q < G; ++q) {
      auto& rk = pl->ranks[q];
      CUDA_TRY(cudaSetDevice(rk.dev));
      // the copy stream starts where the rank's stream is (behind every rank's previous work)
      CUDA_TRY(cudaEventRecord(rk.ev, S(q)));
      CUDA_TRY(cudaStreamWaitEvent(CS(q), rk.ev, 0));
      CUDA_TRY(cudaStreamWaitEvent(CO(q), rk.ev, 0));
      for (int i = 0; i < C; ++i) {  // exchange 1, column chunk i: B_q[p L1 + r][i c2 + c] = x_p[r][q L2 + i c2 + c]
        for (int p = 0; p < G; ++p)
          CUDA_TRY(cudaMemcpy2DAsync(W(q) + (size_t)(p * L1 * L2 + i * c2) * e, L2 * e,
                                     (const char*)in[p] + (size_t)(q * L2 + i * c2) * e, N2 * e, c2 * e, L1,
                                     cudaMemcpyDefault, CS(q)));
        CUDA_TRY(cudaEventRecord(EV(q, 0, i), CS(q)));
      }
      for (int i = 0; i < C; ++i) {  // pass 1, chunk i: columns [i c2, (i+1) c2) -> rows of Y'_q (in out_q)
        CUDA_TRY(cudaStreamWaitEvent(S(q), EV(q, 0, i), 0));
        CUDA_TRY(cudaMemsetAsync(rk.lp[0].a.ctr, 0, (size_t)rk.lp[0].counter_ints * 4, S(q)));
        rc = launch_lean(rk.lp[0], W(q) + (size_t)(i * c2) * e, (char*)out[q] + (size_t)(i * c2 * N1) * e, S(q), i * c2);
        if (rc != EFFT_OK) return rc;
        CUDA_TRY(cudaEventRecord(EV(q, 1, i), S(q)));
      }
      for (int i = 0; i < C; ++i) {  // exchange 2, slab i (pushed): T_p[q L2 + i c2 + c][k1'] = Y'_q[i c2 + c][p L1 + k1']
        CUDA_TRY(cudaStreamWaitEvent(CO(q), EV(q, 1, i), 0));
        for (int p = 0; p < G; ++p)
          CUDA_TRY(cudaMemcpy2DAsync(W2(p) + (size_t)((q * L2 + i * c2) * L1) * e, L1 * e,
                                     (const char*)out[q] + (size_t)(i * c2 * N1 + p * L1) * e, N1 * e, L1 * e, c2,
                                     cudaMemcpyDefault, CO(q)));
        CUDA_TRY(cudaEventRecord(EV(q, 2, i), CO(q)));
      }
    }
    for (int p = 0; p < G; ++p) {
      auto& rk = pl->ranks[p];
      CUDA_TRY(cudaSetDevice(rk.dev));
      for (int q = 0; q < G; ++q)
        for (int i = 0; i < C; ++i) CUDA_TRY(cudaStreamWaitEvent(S(p), EV(q, 2, i), 0));
      for (int j = 0; j < C; ++j) {  // pass 2 in place on T_p, column chunk j
        CUDA_TRY(cudaMemsetAsync(rk.lp[1].a.ctr, 0, (size_t)rk.lp[1].counter_ints * 4, S(p)));
        rc = launch_lean(rk.lp[1], W2(p) + (size_t)(j * c1) * e, W2(p) + (size_t)(j * c1) * e, S(p));
        if (rc != EFFT_OK) return rc;
        CUDA_TRY(cudaEventRecord(EV(p, 3, j), S(p)));
        // exchange 3, slab j (pushed): y_r[k2'][p L1 + j c1 + k1'] = X_p[r L2 + k2'][j c1 + k1'].  out_r is free:
        // pass 2 anywhere implies every rank's exchange 2 has left it
        CUDA_TRY(cudaStreamWaitEvent(CO(p), EV(p, 3, j), 0));
        for (int r = 0; r < G; ++r)
          CUDA_TRY(cudaMemcpy2DAsync((char*)out[r] + (size_t)(p * L1 + j * c1) * e, N1 * e,
                                     W2(p) + (size_t)(r * L2 * L1 + j * c1) * e, L1 * e, c1 * e, L2, cudaMemcpyDefault,
                                     CO(p)));
        CUDA_TRY(cudaEventRecord(EV(p, 4, j), CO(p)));
      }
    }
    for (int r = 0; r < G; ++r) {  // every rank's stream ends behind every exchange-3 slab
      CUDA_TRY(cudaSetDevice(pl->ranks[r].dev));
      for (int p = 0; p < G; ++p)
        for (int j = 0; j < C; ++j) CUDA_TRY(cudaStreamWaitEvent(S(r), EV(p, 4, j), 0));
    }
    return all_wait();
  }
  // exchange 1 (pulled by the destination): B_q[p L1 + r][c] = x_p[r][q L2 + c]
  for (int q = 0; q < G; ++q) {
    CUDA_TRY(cudaSetDevice(pl->ranks[q].dev));
    for (int p = 0; p < G; ++p)
      CUDA_TRY(cudaMemcpy2DAsync(W(q) + (size_t)(p * L1 * L2) * e, L2 * e, (const char*)in[p] + (size_t)(q * L2) * e,
                                 N2 * e, L2 * e, L1, cudaMemcpyDefault, S(q)));
    // pass 1: B_q -> Y'_q[c][k1] (in out_q), twiddle W_N^((q L2 + c) k1)
    CUDA_TRY(cudaMemsetAsync(pl->ranks[q].counters, 0, pl->ranks[q].counter_bytes, S(q)));
    rc = launch_lean(pl->ranks[q].lp[0], W(q), out[q], S(q));
    if (rc != EFFT_OK) return rc;
  }
  rc = all_wait();
  if (rc != EFFT_OK) return rc;
  // exchange 2: T_p[q L2 + c][k1'] = Y'_q[c][p L1 + k1']; pass 2 in place on T_p
  for (int p = 0; p < G; ++p) {
    CUDA_TRY(cudaSetDevice(pl->ranks[p].dev));
    for (int q = 0; q < G; ++q)
      CUDA_TRY(cudaMemcpy2DAsync(W(p) + (size_t)(q * L2 * L1) * e, L1 * e, (const char*)out[q] + (size_t)(p * L1) * e,
                                 N1 * e, L1 * e, L2, cudaMemcpyDefault, S(p)));
    rc = launch_lean(pl->ranks[p].lp[1], W(p), W(p), S(p));
    if (rc != EFFT_OK) return rc;
  }
  rc = all_wait();
  if (rc != EFFT_OK) return rc;
  // exchange 3: y_r[k2'][p L1 + k1'] = X_p[r L2 + k2'][k1'] (natural-order output blocks)
  for (int r = 0; r < G; ++r) {
    CUDA_TRY(cudaSetDevice(pl->ranks[r].dev));
    for (int p = 0; p < G; ++p)
      CUDA_TRY(cudaMemcpy2DAsync((char*)out[r] + (size_t)(p * L1) * e, N1 * e, W(p) + (size_t)(r * L2 * L1) * e,
                                 L1 * e, L1 * e, L2, cudaMemcpyDefault, S(r)));
  }
  // the exchange-3 sources (work arrays) are reused by the next call only
  // after every rank's stream has passed this point
  return all_wait();
}

int efft_plan_create_shard_rank(efft_plan_t* out, int64_t n, int dtype, int direction, int ngpus, int rank,
                                int device, uint32_t flags) {
  if (!out) return fail(EFFT_ERR_INVALID_ARG, "plan pointer is NULL");
  *out = nullptr;
  if (dtype != EFFT_C64 && dtype != EFFT_C128) return fail(EFFT_ERR_INVALID_ARG, "dtype %d (complex only)", dtype);
  if (direction != EFFT_FORWARD && direction != EFFT_INVERSE)
    return fail(EFFT_ERR_INVALID_ARG, "direction must be -1 or +1, got %d", direction);
  if (ngpus < 2 || ngpus > 64 || (ngpus & (ngpus - 1)) || rank < 0 || rank >= ngpus)
    return fail(EFFT_ERR_INVALID_ARG, "ngpus must be a power of two in [2, 64], 0 <= rank < ngpus");
  const int c128 = dtype == EFFT_C128;
  int64_t N1, N2;
  if (!efft::lean::split_sharded(n, ngpus, c128, &N1, &N2))
    return fail(EFFT_ERR_UNSUPPORTED_SIZE, "n=%lld cannot be sharded over %d ranks", (long long)n, ngpus);
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(EFFT_ERR_INVALID_ARG, "device %d of %d", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  efft_plan_s* pl = new efft_plan_s();
  pl->n = pl->n_user = n;
  pl->dtype = dtype;
  pl->direction = direction;
  pl->device = device;
  pl->flags = flags;
  pl->elem = c128 ? 16 : 8;
  pl->npass = 2;
  pl->sh_n1 = N1;
  pl->sh_n2 = N2;
  pl->sh_rank = rank;
  pl->sh_world = ngpus;
  pl->ranks.resize(1);
  auto& r = pl->ranks[0];
  r.dev = device;
  int sms = 0, ecuda = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int64_t stg = 0;
  if (!efft::lean::plan_sharded(n, ngpus, rank, c128, direction == EFFT_INVERSE, (flags & EFFT_FLAG_CHECK_FINITE) != 0,
                                sms, r.lp, &stg, &ecuda, true)) {
    efft_plan_destroy(pl);
    return ecuda ? fail(EFFT_ERR_CUDA, "shard pass setup failed") : fail(EFFT_ERR_UNSUPPORTED_SIZE, "no pass kernel");
  }
  r.counter_bytes = (size_t)(r.lp[0].counter_ints + r.lp[1].counter_ints) * 4;
  if (cudaMalloc(&r.staging, (size_t)stg * pl->elem) != cudaSuccess ||
      cudaMalloc((void**)&r.counters, r.counter_bytes) != cudaSuccess || cudaMalloc((void**)&r.flag, 4) != cudaSuccess ||
      cudaMemset(r.flag, 0, 4) != cudaSuccess) {
    cudaGetLastError();
    efft_plan_destroy(pl);
    return fail(EFFT_ERR_ALLOC, "shard rank buffers");
  }
  int64_t off = 0;
  for (auto& ps : r.lp) {
    ps.a.stg = r.staging;
    ps.a.ctr = reinterpret_cast<unsigned long long*>(r.counters + off);
    ps.a.doneA = r.counters + off + 2;
    ps.a.doneB = ps.a.doneA + ps.a.ngroups;
    ps.a.flag = r.flag;
    off += ps.counter_ints;
  }
  *out = pl;
  return EFFT_OK;
}

int efft_execute_shard_pass(efft_plan_t pl, int pass, const void* in, void* out, void* stream) {
  if (!pl || !in || !out || pl->ranks.size() != 1 || pl->sh_world < 2)
    return fail(EFFT_ERR_INVALID_ARG, "not a shard-rank plan or NULL buffer");
  if (pass != 0 && pass != 1) return fail(EFFT_ERR_INVALID_ARG, "pass must be 0 or 1");
  if (pass == 0 && in == out) return fail(EFFT_ERR_INVALID_ARG, "pass 0 cannot run in place");
  auto& r = pl->ranks[0];
  CUDA_TRY(cudaSetDevice(r.dev));
  cudaStream_t s = (cudaStream_t)stream;
  efft::lean::Pass& q = r.lp[pass];
  CUDA_TRY(cudaMemsetAsync(q.a.ctr, 0, (size_t)q.counter_ints * 4, s));
  return launch_lean(q, in, out, s);
}

int efft_sharded_split(efft_plan_t pl, int64_t* n1, int64_t* n2) {
  if (!pl || !n1 || !n2 || pl->ranks.empty()) return fail(EFFT_ERR_INVALID_ARG, "not a sharded plan");
  *n1 = pl->sh_n1;
  *n2 = pl->sh_n2;
  return EFFT_OK;
}

int efft_plan_destroy(efft_plan_t pl) {
  if (!pl) return EFFT_OK;
  for (auto& r : pl->ranks) {
    cudaSetDevice(r.dev);
    if (r.staging) cudaFree(r.staging);
    if (r.counters) cudaFree(r.counters);
    if (r.flag) cudaFree(r.flag);
    if (r.work) cudaFree(r.work);
    if (r.work2) cudaFree(r.work2);
    if (r.cs) cudaStreamDestroy(r.cs);
    if (r.cs2) cudaStreamDestroy(r.cs2);
    for (auto& e : r.cev)
      if (e) cudaEventDestroy(e);
    if (r.ev) cudaEventDestroy(r.ev);
  }
  cudaSetDevice(pl->device);
  for (auto& e : pl->tev)
    if (e) cudaEventDestroy(e);
  if (pl->staging) cudaFree(pl->staging);
  if (pl->counters) cudaFree(pl->counters);
  if (pl->flag) cudaFree(pl->flag);
  delete pl;
  return EFFT_OK;
}

}  // extern "C"

/*
 * efft_oracle.c -- CPU restatement of the reference EFFT algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1409_5757_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker or as the
 * timed CPU baseline.  The product path fails loudly without its CUDA library.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks this restatement against
 * the reference's own known-answer vectors (pkg/tests/test_leaf_dft.py:22-38,
 * test_recombine.py:40-63, test_oracle.py:12-24, test_scatter.py:40-48) and
 * against golden fixtures produced by importing the reference package
 * (tests/golden/make_golden.py -> tests/golden/ fixtures).
 *
 * The reference (pkg/src/efft) is real-input float32 only.  This restatement
 * keeps its three stages and equations but runs them on complex data, which is
 * the form BASELINE.json's configs need:
 *
 *   Stage I   scatter   : element i*b + j -> bin bitrev_s(j), offset i
 *                         (scatter.py:18-28, 31-57)
 *   Stage II  leaf      : per-bin radix-2 DIT -- bit-reverse gather, then
 *                         log2 stages with W = exp(-i*pi*j/half)
 *                         (leaf_dft.py:32-39, 42-68, 93-111; the real split of
 *                         leaf_dft.py:113-125 is not needed for complex data).
 *                         Bins of size M*2^t (M = 3) end in a direct M-point DFT
 *                         with an exact integer phase (oracle.py:35-53), the
 *                         M x 2^s extension of PAPER.md:85, 191.
 *   Stage III merge     : s levels of F_k = E_k + W_k O_k, F_{k+m} = E_k - W_k O_k,
 *                         W_k = exp(-i*pi*k/m)  (recombine.py:79-105, 216-260)
 *
 * Two precisions:
 *   efo_transform_c128 -- fp64 data, twiddles from exact integer index in fp64.
 *                         This is the parity ground truth.
 *   efo_transform_c64  -- float32 data with the reference's own twiddle recipe:
 *                         angle formed in fp64, rounded to float32, float32
 *                         cos/sin (recombine.py:49-59), stage tables rounded
 *                         from fp64 to complex64 (leaf_dft.py:55-58).  This is
 *                         the reference-precision CPU path timed by bench.py.
 * Inverse (direction = +1): conjugate twiddles and 1/N scale (not in the
 * reference; added for BASELINE.json configs 2 and 5).
 *
 * efo_dft_at is the O(N) direct sum of oracle.py:79-89 for complex input:
 * exact (k*n) mod N phase, fp64 accumulation in fixed 2^16 chunks.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EFO_OK 0
#define EFO_EINVAL 1
#define EFO_ENOMEM 2

static const double EFO_PI = 3.14159265358979323846264338327950288;

int efo_version(void) { return 1; }

/* scatter.py:18-28 -- s-bit bit reversal (an involution). */
int64_t efo_bitrev(int64_t j, int bits) {
  int64_t r = 0;
  for (int b = 0; b < bits; ++b) {
    r = (r << 1) | (j & 1);
    j >>= 1;
  }
  return r;
}

/* Size decomposition n = M * 2^t with M odd in {1, 3, 5, 7}. */
static int efo_factor(int64_t n, int64_t *M, int *t) {
  if (n < 1) return EFO_EINVAL;
  int tt = 0;
  while ((n & 1) == 0) {
    n >>= 1;
    ++tt;
  }
  if (n != 1 && n != 3 && n != 5 && n != 7) return EFO_EINVAL;
  *M = n;
  *t = tt;
  return EFO_OK;
}

static void efo_set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

/* ---------------------------------------------------------------------------
 * The body below is instantiated twice (REAL = double / float).
 * ------------------------------------------------------------------------- */

#define EFO_DEFINE(SUF, REAL, TWIDDLE)                                          \
  /* Stage I: scatter.py:31-57, dst[bitrev(j)*m + i] = src[i*b + j]. */         \
  static void efo_scatter_##SUF(const REAL *x, REAL *y, int64_t n, int s,       \
                                int conj_in) {                                  \
    int64_t b = (int64_t)1 << s, m = n >> s;                                    \
    _Pragma("omp parallel for schedule(static)")                                \
    for (int64_t j = 0; j < b; ++j) {                                           \
      int64_t dst = efo_bitrev(j, s) * m;                                       \
      for (int64_t i = 0; i < m; ++i) {                                         \
        y[2 * (dst + i)] = x[2 * (i * b + j)];                                  \
        y[2 * (dst + i) + 1] =                                                  \
            conj_in ? -x[2 * (i * b + j) + 1] : x[2 * (i * b + j) + 1];         \
      }                                                                         \
    }                                                                           \
  }                                                                             \
                                                                                \
  /* One radix-2 merge of two adjacent half-spectra of length h, in place:    \
   * recombine.py:79-105 in complex form, W_k = exp(-i*pi*k/h). */              \
  static void efo_merge_##SUF(REAL *seg, int64_t h, const REAL *tw) {           \
    REAL *e = seg, *o = seg + 2 * h;                                            \
    for (int64_t k = 0; k < h; ++k) {                                           \
      REAL wr = tw[2 * k], wi = tw[2 * k + 1];                                  \
      REAL orr = o[2 * k], oi = o[2 * k + 1];                                   \
      REAL tr = orr * wr - oi * wi;                                             \
      REAL ti = orr * wi + oi * wr;                                             \
      REAL er = e[2 * k], ei = e[2 * k + 1];                                    \
      e[2 * k] = er + tr;                                                       \
      e[2 * k + 1] = ei + ti;                                                   \
      o[2 * k] = er - tr;                                                       \
      o[2 * k + 1] = ei - ti;                                                   \
    }                                                                           \
  }                                                                             \
                                                                                \
  /* Direct M-point DFT of a bin base (M = 3), exact integer phase as in      \
   * oracle.py:43-51. */                                                        \
  static void efo_small_dft_##SUF(REAL *v, int64_t M) {                         \
    if (M == 1) return;                                                         \
    double tmp[2 * 7]; /* M <= 7 */                                             \
    for (int64_t k = 0; k < M; ++k) {                                           \
      double ar = 0, ai = 0;                                                    \
      for (int64_t n = 0; n < M; ++n) {                                         \
        int64_t r = (k * n) % M;                                                \
        double c = cos(-2.0 * EFO_PI * (double)r / (double)M);                  \
        double sn = sin(-2.0 * EFO_PI * (double)r / (double)M);                 \
        ar += (double)v[2 * n] * c - (double)v[2 * n + 1] * sn;                 \
        ai += (double)v[2 * n] * sn + (double)v[2 * n + 1] * c;                 \
      }                                                                         \
      tmp[2 * k] = ar;                                                          \
      tmp[2 * k + 1] = ai;                                                      \
    }                                                                           \
    for (int64_t k = 0; k < 2 * M; ++k) v[k] = (REAL)tmp[k];                    \
  }                                                                             \
                                                                                \
  /* Stage II: leaf_dft.py:93-111 (complex part of the leaf): bit-reverse     \
   * gather of 2^t blocks of M, M-point base DFTs, t radix-2 stages. */         \
  static void efo_leaf_##SUF(REAL *bin, int64_t len, int64_t M, REAL *work,     \
                             const REAL *const *stage_tw) {                     \
    int64_t p = len / M;                                                        \
    int t = 0;                                                                  \
    while (((int64_t)1 << t) < p) ++t;                                          \
    for (int64_t j = 0; j < p; ++j) {                                           \
      int64_t jr = efo_bitrev(j, t);                                            \
      for (int64_t i = 0; i < M; ++i) {                                         \
        work[2 * (jr * M + i)] = bin[2 * (i * p + j)];                          \
        work[2 * (jr * M + i) + 1] = bin[2 * (i * p + j) + 1];                  \
      }                                                                         \
    }                                                                           \
    for (int64_t j = 0; j < p; ++j) efo_small_dft_##SUF(work + 2 * j * M, M);   \
    int lvl = 0;                                                                \
    for (int64_t h = M; h < len; h *= 2, ++lvl)                                 \
      for (int64_t s0 = 0; s0 < len; s0 += 2 * h)                               \
        efo_merge_##SUF(work + 2 * s0, h, stage_tw[lvl]);                       \
    memcpy(bin, work, sizeof(REAL) * 2 * len);                                  \
  }                                                                             \
                                                                                \
  static void efo_fill_tw_##SUF(REAL *tw, int64_t h, int64_t k0, int64_t cnt,   \
                                int inverse) {                                  \
    for (int64_t k = 0; k < cnt; ++k) {                                         \
      REAL c, sn;                                                               \
      TWIDDLE(k0 + k, h, c, sn);                                                \
      tw[2 * k] = c;                                                            \
      tw[2 * k + 1] = inverse ? -sn : sn;                                       \
    }                                                                           \
  }                                                                             \
                                                                                \
  int efo_transform_##SUF(int64_t n, int splits, const REAL *x, REAL *y,        \
                          int direction, int threads) {                         \
    int64_t M;                                                                  \
    int t;                                                                      \
    if (efo_factor(n, &M, &t) != EFO_OK) return EFO_EINVAL;                     \
    if (splits < 0 || splits > t) return EFO_EINVAL;                            \
    if (direction != -1 && direction != 1) return EFO_EINVAL;                   \
    efo_set_threads(threads);                                                   \
    int inverse = direction == 1;                                               \
    int s = splits;                                                             \
    int64_t m = n >> s;                                                         \
    /* conj(F(conj(x))) == inverse DFT (unscaled). */                           \
    efo_scatter_##SUF(x, y, n, s, inverse);                                     \
    /* Per-stage leaf tables (leaf_dft.py:52-58): one per radix-2 level. */     \
    int nl = 0;                                                                 \
    for (int64_t h = M; h < m; h *= 2) ++nl;                                    \
    REAL **stage_tw = (REAL **)calloc((size_t)(nl + 1), sizeof(REAL *));        \
    if (!stage_tw) return EFO_ENOMEM;                                           \
    {                                                                           \
      int lvl = 0;                                                              \
      for (int64_t h = M; h < m; h *= 2, ++lvl) {                               \
        stage_tw[lvl] = (REAL *)malloc(sizeof(REAL) * 2 * (size_t)h);           \
        if (!stage_tw[lvl]) return EFO_ENOMEM;                                  \
        efo_fill_tw_##SUF(stage_tw[lvl], h, 0, h, 0);                           \
      }                                                                         \
    }                                                                           \
    int64_t bins = (int64_t)1 << s;                                             \
    int failed = 0;                                                             \
    _Pragma("omp parallel")                                                     \
    {                                                                           \
      REAL *work = (REAL *)malloc(sizeof(REAL) * 2 * (size_t)m);                \
      if (!work) {                                                              \
        _Pragma("omp atomic write") failed = 1;                                 \
      } else {                                                                  \
        _Pragma("omp for schedule(dynamic, 1)")                                 \
        for (int64_t bi = 0; bi < bins; ++bi)                                   \
          efo_leaf_##SUF(y + 2 * bi * m, m, M, work, (const REAL *const *)stage_tw); \
        free(work);                                                             \
      }                                                                         \
    }                                                                           \
    for (int lvl = 0; lvl < nl; ++lvl) free(stage_tw[lvl]);                     \
    free(stage_tw);                                                             \
    if (failed) return EFO_ENOMEM;                                              \
    /* Stage III: s merge levels (recombine.py:263-295 without recursion).      \
     * Twiddles are generated in k-blocks so memory stays O(threads*block). */  \
    const int64_t KB = 4096;                                                    \
    for (int64_t h = m; h < n; h *= 2) {                                        \
      int64_t nseg = n / (2 * h);                                               \
      int64_t nkb = (h + KB - 1) / KB;                                          \
      _Pragma("omp parallel")                                                   \
      {                                                                         \
        REAL *tw = (REAL *)malloc(sizeof(REAL) * 2 * (size_t)KB);               \
        _Pragma("omp for schedule(dynamic, 1)")                                 \
        for (int64_t kb = 0; kb < nkb; ++kb) {                                  \
          int64_t k0 = kb * KB, cnt = (h - k0) < KB ? (h - k0) : KB;            \
          efo_fill_tw_##SUF(tw, h, k0, cnt, 0);                                 \
          for (int64_t sg = 0; sg < nseg; ++sg) {                               \
            REAL *e = y + 2 * (sg * 2 * h + k0);                                \
            REAL *o = e + 2 * h;                                                \
            for (int64_t k = 0; k < cnt; ++k) {                                 \
              REAL wr = tw[2 * k], wi = tw[2 * k + 1];                          \
              REAL orr = o[2 * k], oi = o[2 * k + 1];                           \
              REAL tr = orr * wr - oi * wi, ti = orr * wi + oi * wr;            \
              REAL er = e[2 * k], ei = e[2 * k + 1];                            \
              e[2 * k] = er + tr;                                               \
              e[2 * k + 1] = ei + ti;                                           \
              o[2 * k] = er - tr;                                               \
              o[2 * k + 1] = ei - ti;                                           \
            }                                                                   \
          }                                                                     \
        }                                                                       \
        free(tw);                                                               \
      }                                                                         \
    }                                                                           \
    if (inverse) {                                                              \
      REAL sc = (REAL)(1.0 / (double)n);                                        \
      _Pragma("omp parallel for schedule(static)")                              \
      for (int64_t i = 0; i < n; ++i) {                                         \
        y[2 * i] *= sc;                                                         \
        y[2 * i + 1] = -y[2 * i + 1] * sc;                                      \
      }                                                                         \
    }                                                                           \
    return EFO_OK;                                                              \
  }

/* fp64 twiddle: exact integer index k < h, W = exp(-i*pi*k/h) evaluated in
 * fp64 (oracle.py:43-51 style: integer phase, then one fp64 scaling). */
#define EFO_TW64(k, h, c, s)                                                    \
  do {                                                                          \
    double a_ = -EFO_PI * (double)(k) / (double)(h);                            \
    c = cos(a_);                                                                \
    s = sin(a_);                                                                \
  } while (0)

/* Reference twiddle recipe (recombine.py:49-59): angle formed in fp64,
 * rounded to float32, float32 cos/sin. */
#define EFO_TW32(k, h, c, s)                                                    \
  do {                                                                          \
    float a_ = (float)((double)(k) * (-EFO_PI / (double)(h)));                  \
    c = cosf(a_);                                                               \
    s = sinf(a_);                                                               \
  } while (0)

EFO_DEFINE(c128, double, EFO_TW64)
EFO_DEFINE(c64, float, EFO_TW32)

/* oracle.py:79-89 for complex input: one coefficient, O(N), exact phase.
 * The phase index (k*i) mod n is exact in integers; the root is formed as
 * W^((k*B*h) mod n) * W^((k*l) mod n) for i = h*B + l, both factors from fp64
 * cos/sin of an exact integer index, so each term carries ~1 ulp of phase
 * error (oracle.py:43-51 evaluates one exp per term; this is the same value to
 * rounding, ~100x cheaper).  Accumulation in fixed 2^16-element chunks. */
void efo_dft_at(int64_t n, const double *x, int64_t k, int direction,
                double *out2) {
  const int64_t B = 4096;
  double sgn = direction == 1 ? 1.0 : -1.0;
  int64_t kk = ((k % n) + n) % n;
  double *tl = (double *)malloc(sizeof(double) * 2 * (size_t)B);
  for (int64_t l = 0; l < B; ++l) {
    unsigned __int128 e = (unsigned __int128)kk * (unsigned __int128)l;
    int64_t r = (int64_t)(e % (unsigned __int128)n);
    double a = sgn * 2.0 * EFO_PI * ((double)r / (double)n);
    tl[2 * l] = cos(a);
    tl[2 * l + 1] = sin(a);
  }
  double tr = 0, ti = 0, cr = 0, ci = 0;
  for (int64_t h = 0; h * B < n; ++h) {
    unsigned __int128 e = (unsigned __int128)kk * (unsigned __int128)(h * B);
    int64_t r = (int64_t)(e % (unsigned __int128)n);
    double a = sgn * 2.0 * EFO_PI * ((double)r / (double)n);
    double hr = cos(a), hi = sin(a);
    int64_t lim = n - h * B < B ? n - h * B : B;
    const double *xp = x + 2 * h * B;
    for (int64_t l = 0; l < lim; ++l) {
      double wr = hr * tl[2 * l] - hi * tl[2 * l + 1];
      double wi = hr * tl[2 * l + 1] + hi * tl[2 * l];
      cr += xp[2 * l] * wr - xp[2 * l + 1] * wi;
      ci += xp[2 * l] * wi + xp[2 * l + 1] * wr;
    }
    if (((h + 1) * B) % ((int64_t)1 << 16) == 0) {
      tr += cr;
      ti += ci;
      cr = ci = 0;
    }
  }
  tr += cr;
  ti += ci;
  free(tl);
  out2[0] = tr;
  out2[1] = ti;
}

/* Many spot coefficients in parallel (one per thread). */
void efo_dft_at_many(int64_t n, const double *x, const int64_t *ks, int64_t nk,
                     int direction, double *out, int threads) {
  efo_set_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nk; ++q) efo_dft_at(n, x, ks[q], direction, out + 2 * q);
}

/* Batched strided sub-FFT pass with a fused DIT twiddle -- the CPU mirror of
 * the device pass contract (include/efft_b200.h: efft_pass_desc), used by the
 * sharded host logic tests.  For every column c in [0, cols) and batch item
 * g in [0, batch):
 *   v[r]   = in[g*in_batch + c*in_col + r*in_stride]        r in [0, len)
 *   v[r]  *= exp(sign*2*pi*i * ((tw_base + c*tw_col + g*tw_batch) * r mod tw_mod) / tw_mod)
 *            (skipped when tw_mod == 0)
 *   out[g*out_batch + c*out_col + k*out_stride] = sum_r v[r] exp(sign*2*pi*i*k*r/len)
 * sign = -1 forward, +1 inverse (unscaled).  fp64 complex, direct O(len^2)
 * per column for len <= 64, else the restated radix-2 transform above. */
int efo_pass_c128(const double *in, double *out, int64_t len, int64_t cols,
                  int64_t batch, int64_t in_col, int64_t in_stride,
                  int64_t in_batch, int64_t out_col, int64_t out_stride,
                  int64_t out_batch, int64_t tw_mod, int64_t tw_base,
                  int64_t tw_col, int64_t tw_batch, int direction, int threads) {
  int64_t M;
  int t;
  if (efo_factor(len, &M, &t) != EFO_OK) return EFO_EINVAL;
  efo_set_threads(threads);
  double sgn = direction == 1 ? 1.0 : -1.0;
  int failed = 0;
#pragma omp parallel
  {
    double *v = (double *)malloc(sizeof(double) * 2 * (size_t)len);
    double *w = (double *)malloc(sizeof(double) * 2 * (size_t)len);
    if (!v || !w) {
#pragma omp atomic write
      failed = 1;
    } else {
#pragma omp for collapse(2) schedule(dynamic, 16)
      for (int64_t g = 0; g < batch; ++g)
        for (int64_t c = 0; c < cols; ++c) {
          const double *src = in + 2 * (g * in_batch + c * in_col);
          for (int64_t r = 0; r < len; ++r) {
            double vr = src[2 * r * in_stride], vi = src[2 * r * in_stride + 1];
            if (tw_mod > 0) {
              int64_t a = tw_base + c * tw_col + g * tw_batch;
              unsigned __int128 e = (unsigned __int128)(a % tw_mod) * (unsigned __int128)r;
              int64_t em = (int64_t)(e % (unsigned __int128)tw_mod);
              double ang = sgn * 2.0 * EFO_PI * (double)em / (double)tw_mod;
              double cr = cos(ang), ci = sin(ang);
              double tr = vr * cr - vi * ci;
              vi = vr * ci + vi * cr;
              vr = tr;
            }
            /* forward transform of conj(v) then conj gives the inverse */
            v[2 * r] = vr;
            v[2 * r + 1] = direction == 1 ? -vi : vi;
          }
          efo_transform_c128(len, 0, v, w, -1, 1);
          double *dst = out + 2 * (g * out_batch + c * out_col);
          for (int64_t k = 0; k < len; ++k) {
            dst[2 * k * out_stride] = w[2 * k];
            dst[2 * k * out_stride + 1] = direction == 1 ? -w[2 * k + 1] : w[2 * k + 1];
          }
        }
    }
    free(v);
    free(w);
  }
  return failed ? EFO_ENOMEM : EFO_OK;
}

/*
 * oracle/nq_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * NanoQuant reference algorithm for the binary low-rank hot path.
 *
 * It exists so the parity checks do not depend on the reference build: every
 * function below restates the reference function it names (file:line under
 * /root/reference/proj) with the SAME floating-point operation order, so that
 * compiled with the reference's flags (-O3, no -march, no -ffast-math; x86-64
 * therefore never contracts to FMA) it is bit-identical to the reference.
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   - the reference's own known-answer vectors (test_packed.cpp, test_linalg.cpp,
 *     test_admm.cpp, test_balance.cpp, test_storage.cpp), and
 *   - bitwise comparison against oracle/_ref/libnqref.so, the unmodified
 *     reference library compiled from /root/reference by oracle/Makefile,
 *     plus the committed fixtures under tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path (paper_2602_06694_b200) never does.
 * Status codes follow include/nqb.h.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/nqb.h"

/* ------------------------------------------------------------------------ */
/* splitmix64 Rng (rng.hpp:25-58)                                            */
/* ------------------------------------------------------------------------ */
typedef struct { uint64_t state; } nqo_rng;

static uint64_t rng_next(nqo_rng* r) { /* rng.hpp:29-34 */
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static double rng_uniform(nqo_rng* r) { /* rng.hpp:37-39 */
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
static double rng_gaussian(nqo_rng* r) { /* rng.hpp:44-49 */
  double u1 = rng_uniform(r);
  while (u1 <= 0.0) u1 = rng_uniform(r);
  const double u2 = rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void* nqo_rng_create(uint64_t seed) {
  nqo_rng* r = (nqo_rng*)malloc(sizeof(nqo_rng));
  r->state = seed;
  return r;
}
void nqo_rng_destroy(void* h) { free(h); }
void nqo_rng_u64(void* h, uint64_t count, uint64_t* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_next((nqo_rng*)h);
}
void nqo_rng_uniform(void* h, double lo, double hi, uint64_t count, double* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * rng_uniform((nqo_rng*)h);
}
void nqo_rng_gaussian(void* h, uint64_t count, double* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_gaussian((nqo_rng*)h);
}
void nqo_rng_sign(void* h, uint64_t count, double* out) { /* rng.hpp:54 */
  for (uint64_t i = 0; i < count; ++i) out[i] = (rng_next((nqo_rng*)h) & 1u) ? 1.0 : -1.0;
}
void nqo_rng_index(void* h, uint64_t n, uint64_t count, uint64_t* out) { /* rng.hpp:52 */
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_next((nqo_rng*)h) % n;
}

/* ------------------------------------------------------------------------ */
/* binary16 (half.hpp:26-89)                                                 */
/* ------------------------------------------------------------------------ */
static uint16_t float_to_half(float value) { /* half.hpp:26-56 */
  uint32_t bits;
  memcpy(&bits, &value, 4);
  const uint32_t sign = (bits >> 16) & 0x8000u;
  const int32_t exponent = (int32_t)((bits >> 23) & 0xFFu) - 127;
  uint32_t mantissa = bits & 0x7FFFFFu;
  if (exponent == 128) return (uint16_t)(sign | 0x7C00u | (mantissa ? 0x200u : 0u));
  if (exponent > 15) return (uint16_t)(sign | 0x7C00u);
  if (exponent >= -14) {
    uint32_t half = ((uint32_t)(exponent + 15) << 10) | (mantissa >> 13);
    const uint32_t rest = mantissa & 0x1FFFu;
    if (rest > 0x1000u || (rest == 0x1000u && (half & 1u))) ++half;
    return (uint16_t)(sign | half);
  }
  if (exponent >= -25) {
    const uint32_t sig = mantissa | 0x800000u;
    const int shift = -exponent - 1;
    uint32_t half = sig >> shift;
    const uint32_t rest = sig & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    if (rest > halfway || (rest == halfway && (half & 1u))) ++half;
    return (uint16_t)(sign | half);
  }
  return (uint16_t)sign;
}
static float half_to_float(uint16_t h) { /* half.hpp:58-81 */
  const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  const uint32_t exponent = (h >> 10) & 0x1Fu;
  const uint32_t mantissa = h & 0x3FFu;
  uint32_t bits;
  if (exponent == 0x1Fu) {
    bits = sign | 0x7F800000u | (mantissa << 13);
  } else if (exponent != 0) {
    bits = sign | ((exponent + 112u) << 23) | (mantissa << 13);
  } else if (mantissa != 0) {
    uint32_t e = 113, m = mantissa << 13;
    while ((m & 0x800000u) == 0) { m <<= 1; --e; }
    bits = sign | (e << 23) | (m & 0x7FFFFFu);
  } else {
    bits = sign;
  }
  float out;
  memcpy(&out, &bits, 4);
  return out;
}
void nqo_double_to_half(const double* in, uint64_t count, uint16_t* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = float_to_half((float)in[i]);
}
void nqo_half_to_double(const uint16_t* in, uint64_t count, double* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = (double)half_to_float(in[i]);
}

/* ------------------------------------------------------------------------ */
/* Dense core (dense.cpp:21-146)                                             */
/* ------------------------------------------------------------------------ */
typedef struct { size_t rows, cols; double* a; } mat;

static mat mnew(size_t rows, size_t cols) {
  mat m = {rows, cols, (double*)calloc(rows * cols ? rows * cols : 1, sizeof(double))};
  return m;
}
static mat mcopy(const double* p, size_t rows, size_t cols) {
  mat m = mnew(rows, cols);
  memcpy(m.a, p, rows * cols * sizeof(double));
  return m;
}
static void mfree(mat* m) { free(m->a); m->a = NULL; }
#define AT(m, i, j) ((m).a[(i) * (m).cols + (j)])

static int is_finite(const double* p, size_t n) { /* dense.cpp:21-26 */
  for (size_t i = 0; i < n; ++i) if (!isfinite(p[i])) return 0;
  return 1;
}
static int is_zero(const double* p, size_t n) { /* dense.cpp:28-33 */
  for (size_t i = 0; i < n; ++i) if (p[i] != 0.0) return 0;
  return 1;
}
static double sqnorm(const mat* m) { /* dense.cpp:35-39 */
  double s = 0.0;
  for (size_t i = 0; i < m->rows * m->cols; ++i) s += m->a[i] * m->a[i];
  return s;
}
static double fnorm(const mat* m) { return sqrt(sqnorm(m)); } /* dense.cpp:41-43 */
static mat transposed(const mat* m) { /* dense.cpp:46-54 */
  mat t = mnew(m->cols, m->rows);
  for (size_t i = 0; i < m->rows; ++i)
    for (size_t j = 0; j < m->cols; ++j) AT(t, j, i) = AT(*m, i, j);
  return t;
}
static void mscale(mat* m, double f) { /* dense.cpp:56-58 */
  for (size_t i = 0; i < m->rows * m->cols; ++i) m->a[i] *= f;
}
static mat matmul(const mat* a, const mat* b) { /* dense.cpp:60-78 (zero skip) */
  mat c = mnew(a->rows, b->cols);
  for (size_t i = 0; i < a->rows; ++i) {
    double* ci = c.a + i * c.cols;
    const double* ai = a->a + i * a->cols;
    for (size_t k = 0; k < a->cols; ++k) {
      const double aik = ai[k];
      if (aik == 0.0) continue;
      const double* bk = b->a + k * b->cols;
      for (size_t j = 0; j < b->cols; ++j) ci[j] += aik * bk[j];
    }
  }
  return c;
}
static mat matmul_at_b(const mat* a, const mat* b) { /* dense.cpp:80-98 */
  mat c = mnew(a->cols, b->cols);
  for (size_t k = 0; k < a->rows; ++k) {
    const double* ak = a->a + k * a->cols;
    const double* bk = b->a + k * b->cols;
    for (size_t i = 0; i < a->cols; ++i) {
      const double aki = ak[i];
      if (aki == 0.0) continue;
      double* ci = c.a + i * c.cols;
      for (size_t j = 0; j < b->cols; ++j) ci[j] += aki * bk[j];
    }
  }
  return c;
}
static mat madd(const mat* a, const mat* b) { /* dense.cpp:108-115 */
  mat c = mcopy(a->a, a->rows, a->cols);
  for (size_t i = 0; i < c.rows * c.cols; ++i) c.a[i] += b->a[i];
  return c;
}
static mat msub(const mat* a, const mat* b) { /* dense.cpp:117-124 */
  mat c = mcopy(a->a, a->rows, a->cols);
  for (size_t i = 0; i < c.rows * c.cols; ++i) c.a[i] -= b->a[i];
  return c;
}
static double mdot(const mat* a, const mat* b) { /* dense.cpp:132-139 */
  double s = 0.0;
  for (size_t i = 0; i < a->rows * a->cols; ++i) s += a->a[i] * b->a[i];
  return s;
}
static double rel_fro_error(const mat* ref, const mat* approx) { /* dense.cpp:141-146 */
  const double denom = fnorm(ref);
  mat d = msub(ref, approx);
  const double num = fnorm(&d);
  mfree(&d);
  if (denom == 0.0) return num == 0.0 ? 0.0 : INFINITY;
  return num / denom;
}

/* ------------------------------------------------------------------------ */
/* Rank rule (storage.cpp:124-141)                                           */
/* ------------------------------------------------------------------------ */
int nqo_rank_for_target_bpw(uint64_t n, uint64_t m, double t, uint32_t* out) {
  if (n == 0 || m == 0) return NQB_E_VALIDATION;           /* storage.cpp:16-20 */
  if (!(t > 0.0)) return NQB_E_TARGET_TOO_SMALL;
  const double nm = (double)n * (double)m;
  const double ideal = t * nm / (double)(n + m) - 16.0;
  const long long rounded = llround(ideal);
  const uint64_t max_rank = n < m ? n : m;
  if (rounded < 1) {
    const double bpw1 = (double)(1 * (n + m) + 16 * (n + m)) / (double)(n * m); /* :40-47 */
    if (bpw1 > 2.0 * t) return NQB_E_TARGET_TOO_SMALL;
    *out = 1;
    return NQB_OK;
  }
  *out = (uint32_t)((uint64_t)rounded < max_rank ? (uint64_t)rounded : max_rank);
  return NQB_OK;
}

/* ------------------------------------------------------------------------ */
/* Packing (packed.cpp:51-149)                                               */
/* ------------------------------------------------------------------------ */
static size_t wpr_of(size_t cols) { return (cols + 31) / 32; }

int nqo_binarize(const double* in, uint32_t rows, uint32_t cols, double* out) {
  const size_t n = (size_t)rows * cols; /* packed.cpp:51-58 */
  if (!is_finite(in, n)) return NQB_E_NON_FINITE_INPUT;
  for (size_t i = 0; i < n; ++i) out[i] = in[i] < 0.0 ? -1.0 : 1.0;
  return NQB_OK;
}
int nqo_pack_signs(const double* in, uint32_t rows, uint32_t cols, uint32_t* words) {
  const size_t wpr = wpr_of(cols); /* packed.cpp:60-78 */
  memset(words, 0, (size_t)rows * wpr * 4);
  for (size_t i = 0; i < rows; ++i) {
    const double* row = in + i * cols;
    uint32_t* dst = words + i * wpr;
    for (size_t j = 0; j < cols; ++j) {
      if (row[j] == 1.0) dst[j / 32] |= 1u << (j % 32);
      else if (row[j] != -1.0) return NQB_E_NON_BINARY_ENTRY;
    }
  }
  return NQB_OK;
}
int nqo_unpack_signs(const uint32_t* words, uint32_t rows, uint32_t cols, double* out) {
  const size_t wpr = wpr_of(cols); /* packed.cpp:80-103 */
  const uint32_t tail = cols % 32;
  if (tail != 0) {
    const uint32_t pad = ~0u << tail;
    for (size_t i = 0; i < rows; ++i)
      if (words[i * wpr + wpr - 1] & pad) return NQB_E_CORRUPT_PADDING;
  }
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j)
      out[i * cols + j] = (words[i * wpr + j / 32] >> (j % 32)) & 1u ? 1.0 : -1.0;
  return NQB_OK;
}
static int pack_latent(const mat* latent, uint32_t* words) { /* binarize + pack_signs */
  if (!is_finite(latent->a, latent->rows * latent->cols)) return NQB_E_NON_FINITE_INPUT;
  const size_t wpr = wpr_of(latent->cols);
  memset(words, 0, latent->rows * wpr * 4);
  for (size_t i = 0; i < latent->rows; ++i)
    for (size_t j = 0; j < latent->cols; ++j)
      if (!(AT(*latent, i, j) < 0.0)) words[i * wpr + j / 32] |= 1u << (j % 32);
  return NQB_OK;
}
static void reconstruct(uint32_t n, uint32_t m, uint32_t r, const uint32_t* u,
                        const uint32_t* v, const double* s1, const double* s2, double* w) {
  const size_t wpr = wpr_of(r); /* packed.cpp:126-149 */
  const uint32_t tail = r % 32;
  for (size_t i = 0; i < n; ++i) {
    const uint32_t* ur = u + i * wpr;
    for (size_t j = 0; j < m; ++j) {
      const uint32_t* vr = v + j * wpr;
      int64_t agree = 0;
      for (size_t k = 0; k < wpr; ++k) {
        const uint32_t same = ~(ur[k] ^ vr[k]);
        const uint32_t mask = (k + 1 == wpr && tail != 0) ? ((1u << tail) - 1u) : ~0u;
        agree += __builtin_popcount(same & mask);
      }
      const int64_t inner = 2 * agree - (int64_t)r;
      w[i * m + j] = s1[i] * (double)inner * s2[j];
    }
  }
}
int nqo_reconstruct_dense(uint32_t n, uint32_t m, uint32_t r, const uint32_t* u,
                          const uint32_t* v, const double* s1, const double* s2, double* w) {
  reconstruct(n, m, r, u, v, s1, s2, w);
  return NQB_OK;
}

/* gemv_two_stage (packed.cpp:153-192), instantiated for double and float. */
#define GEMV_TWO_STAGE(NAME, ACC)                                                        \
  int NAME(uint32_t n, uint32_t m, uint32_t r, const uint32_t* u, const uint32_t* v,      \
           const double* s1, const double* s2, const ACC* x, uint32_t xlen, ACC* y) {     \
    if (xlen != m) return NQB_E_DIMENSION_MISMATCH;                                      \
    const size_t wpr = wpr_of(r);                                                        \
    ACC* t = (ACC*)calloc(r ? r : 1, sizeof(ACC));                                       \
    for (size_t j = 0; j < m; ++j) {                                                     \
      const ACC a = (ACC)s2[j] * (ACC)x[j];                                              \
      if (a == (ACC)0) continue;                                                         \
      const uint32_t* vr = v + j * wpr;                                                  \
      for (size_t k = 0; k < wpr; ++k) {                                                 \
        uint32_t word = vr[k];                                                           \
        const size_t base = k * 32, lim = (r - base) < 32 ? (r - base) : 32;             \
        for (size_t b = 0; b < lim; ++b) {                                               \
          t[base + b] += (word & 1u) ? a : -a;                                           \
          word >>= 1;                                                                    \
        }                                                                                \
      }                                                                                  \
    }                                                                                    \
    for (size_t i = 0; i < n; ++i) {                                                     \
      const uint32_t* ur = u + i * wpr;                                                  \
      ACC acc = 0;                                                                       \
      for (size_t k = 0; k < wpr; ++k) {                                                 \
        uint32_t word = ur[k];                                                           \
        const size_t base = k * 32, lim = (r - base) < 32 ? (r - base) : 32;             \
        for (size_t b = 0; b < lim; ++b) {                                               \
          acc += (word & 1u) ? t[base + b] : -t[base + b];                               \
          word >>= 1;                                                                    \
        }                                                                                \
      }                                                                                  \
      y[i] = (ACC)s1[i] * acc;                                                           \
    }                                                                                    \
    free(t);                                                                             \
    return NQB_OK;                                                                       \
  }
GEMV_TWO_STAGE(nqo_gemv_f64, double)
GEMV_TWO_STAGE(nqo_gemv_f32, float)

/* gemm_tile / gemm_packed (packed.cpp:210-287); columns are independent and the
 * per-column order equals the reference's, so tiling is irrelevant here. */
int nqo_gemm(uint32_t n, uint32_t m, uint32_t r, const uint32_t* u, const uint32_t* v,
             const double* s1, const double* s2, const double* x, uint32_t b, double* y) {
  const size_t wpr = wpr_of(r);
  double* t = (double*)calloc((size_t)(r ? r : 1) * (b ? b : 1), sizeof(double));
  for (size_t j = 0; j < m; ++j) {
    const double s2j = s2[j];
    const double* xr = x + j * b;
    const uint32_t* vr = v + j * wpr;
    for (size_t k = 0; k < wpr; ++k) {
      uint32_t word = vr[k];
      const size_t base = k * 32, lim = (r - base) < 32 ? (r - base) : 32;
      for (size_t bit = 0; bit < lim; ++bit) {
        double* tr = t + (base + bit) * b;
        if (word & 1u) { for (size_t c = 0; c < b; ++c) tr[c] += s2j * xr[c]; }
        else           { for (size_t c = 0; c < b; ++c) tr[c] -= s2j * xr[c]; }
        word >>= 1;
      }
    }
  }
  double* acc = (double*)calloc(b ? b : 1, sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    const uint32_t* ur = u + i * wpr;
    for (size_t c = 0; c < b; ++c) acc[c] = 0.0;
    for (size_t k = 0; k < wpr; ++k) {
      uint32_t word = ur[k];
      const size_t base = k * 32, lim = (r - base) < 32 ? (r - base) : 32;
      for (size_t bit = 0; bit < lim; ++bit) {
        const double* tr = t + (base + bit) * b;
        if (word & 1u) { for (size_t c = 0; c < b; ++c) acc[c] += tr[c]; }
        else           { for (size_t c = 0; c < b; ++c) acc[c] -= tr[c]; }
        word >>= 1;
      }
    }
    for (size_t c = 0; c < b; ++c) y[i * b + c] = s1[i] * acc[c];
  }
  free(acc);
  free(t);
  return NQB_OK;
}

/* ------------------------------------------------------------------------ */
/* Linear algebra (linalg.cpp:26-239)                                        */
/* ------------------------------------------------------------------------ */
static int try_cholesky(mat* a) { /* linalg.cpp:26-41 */
  const size_t n = a->rows;
  for (size_t j = 0; j < n; ++j) {
    double d = AT(*a, j, j);
    for (size_t k = 0; k < j; ++k) d -= AT(*a, j, k) * AT(*a, j, k);
    if (!(d > 0.0) || !isfinite(d)) return 0;
    const double ljj = sqrt(d);
    AT(*a, j, j) = ljj;
    for (size_t i = j + 1; i < n; ++i) {
      double s = AT(*a, i, j);
      for (size_t k = 0; k < j; ++k) s -= AT(*a, i, k) * AT(*a, j, k);
      AT(*a, i, j) = s / ljj;
    }
  }
  return 1;
}
static mat chol_backsolve(const mat* l, const mat* b) { /* linalg.cpp:44-62 */
  const size_t n = l->rows;
  mat x = mcopy(b->a, b->rows, b->cols);
  for (size_t j = 0; j < b->cols; ++j) {
    for (size_t i = 0; i < n; ++i) {
      double s = AT(x, i, j);
      for (size_t k = 0; k < i; ++k) s -= AT(*l, i, k) * AT(x, k, j);
      AT(x, i, j) = s / AT(*l, i, i);
    }
    for (size_t ii = n; ii-- > 0;) {
      double s = AT(x, ii, j);
      for (size_t k = ii + 1; k < n; ++k) s -= AT(*l, k, ii) * AT(x, k, j);
      AT(x, ii, j) = s / AT(*l, ii, ii);
    }
  }
  return x;
}
static double vnorm(const double* v, size_t n) { /* linalg.cpp:64-68 */
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}
static void vnormalize(double* v, size_t n) { /* linalg.cpp:70-75 */
  const double nn = vnorm(v, n);
  if (nn > 0.0) for (size_t i = 0; i < n; ++i) v[i] /= nn;
}
static void mat_vec(const mat* m, const double* v, double* w) { /* linalg.cpp:78-87 */
  for (size_t i = 0; i < m->rows; ++i) {
    const double* row = m->a + i * m->cols;
    double s = 0.0;
    for (size_t j = 0; j < m->cols; ++j) s += row[j] * v[j];
    w[i] = s;
  }
}
static void mat_t_vec(const mat* m, const double* v, double* w) { /* linalg.cpp:90-99 */
  for (size_t j = 0; j < m->cols; ++j) w[j] = 0.0;
  for (size_t i = 0; i < m->rows; ++i) {
    const double* row = m->a + i * m->cols;
    const double vi = v[i];
    if (vi == 0.0) continue;
    for (size_t j = 0; j < m->cols; ++j) w[j] += row[j] * vi;
  }
}

typedef struct { double sigma; double* left; double* right; int converged; int iters; } pair_t;

static pair_t power_iterate(const mat* m, double* v /* owned */, int max_iters, double tol) {
  pair_t out = {0.0, NULL, NULL, 0, 0}; /* linalg.cpp:101-136 */
  vnormalize(v, m->cols);
  double sigma_prev = -1.0, sigma = 0.0;
  double* mv = (double*)calloc(m->rows ? m->rows : 1, sizeof(double));
  double* w = (double*)calloc(m->cols ? m->cols : 1, sizeof(double));
  int it;
  for (it = 0; it < max_iters; ++it) {
    mat_vec(m, v, mv);
    sigma = vnorm(mv, m->rows);
    if (sigma == 0.0) break;
    mat_t_vec(m, mv, w);
    vnormalize(w, m->cols);
    memcpy(v, w, m->cols * sizeof(double));
    if (sigma_prev >= 0.0 && fabs(sigma - sigma_prev) <= tol * (sigma > 1e-300 ? sigma : 1e-300)) {
      out.converged = 1;
      sigma_prev = sigma;
      ++it;
      break;
    }
    sigma_prev = sigma;
  }
  out.iters = it;
  mat_vec(m, v, mv);
  sigma = vnorm(mv, m->rows);
  out.sigma = sigma;
  out.right = v;
  if (sigma > 0.0) {
    for (size_t i = 0; i < m->rows; ++i) mv[i] /= sigma;
    out.left = mv;
  } else {
    for (size_t i = 0; i < m->rows; ++i) mv[i] = 0.0;
    out.left = mv;
    out.converged = 0;
  }
  free(w);
  return out;
}

static int top_pair(const mat* m, int max_iters, double tol, pair_t* out) {
  if (is_zero(m->a, m->rows * m->cols)) return NQB_E_ZERO_MATRIX; /* linalg.cpp:178-211 */
  double* v0 = (double*)calloc(m->cols ? m->cols : 1, sizeof(double));
  for (size_t i = 0; i < m->rows; ++i) {
    const double* row = m->a + i * m->cols;
    for (size_t j = 0; j < m->cols; ++j) v0[j] += row[j] * row[j];
  }
  for (size_t j = 0; j < m->cols; ++j) v0[j] = sqrt(v0[j]);
  pair_t best = power_iterate(m, v0, max_iters, tol);
  for (size_t j = 0; j < m->cols && best.sigma == 0.0; ++j) { /* :191-198 */
    free(best.left);
    free(best.right);
    double* e = (double*)calloc(m->cols, sizeof(double));
    e[j] = 1.0;
    best = power_iterate(m, e, max_iters, tol);
  }
  size_t arg = 0; /* :200-209 */
  for (size_t j = 1; j < m->cols; ++j)
    if (fabs(best.right[j]) > fabs(best.right[arg])) arg = j;
  if (m->cols > 0 && best.right[arg] < 0.0) {
    for (size_t j = 0; j < m->cols; ++j) best.right[j] = -best.right[j];
    for (size_t i = 0; i < m->rows; ++i) best.left[i] = -best.left[i];
  }
  *out = best;
  return NQB_OK;
}

int nqo_top_singular_pair(const double* a, uint32_t rows, uint32_t cols, int32_t max_iters,
                          double tol, double* sigma, double* left, double* right,
                          int32_t* converged) {
  mat m = {rows, cols, (double*)a};
  pair_t p;
  const int st = top_pair(&m, max_iters, tol, &p);
  if (st) return st;
  *sigma = p.sigma;
  memcpy(left, p.left, rows * sizeof(double));
  memcpy(right, p.right, cols * sizeof(double));
  *converged = p.converged;
  free(p.left);
  free(p.right);
  return NQB_OK;
}

static double spectral_norm(const mat* m, int iters) { /* linalg.cpp:213-216 */
  if (m->rows * m->cols == 0 || is_zero(m->a, m->rows * m->cols)) return 0.0;
  pair_t p = {0.0, NULL, NULL, 0, 0};
  top_pair(m, iters, 1e-14, &p);
  const double s = p.sigma;
  free(p.left);
  free(p.right);
  return s;
}
int nqo_spectral_norm(const double* a, uint32_t rows, uint32_t cols, int32_t iters,
                      double* sigma) {
  mat m = {rows, cols, (double*)a};
  *sigma = spectral_norm(&m, iters);
  return NQB_OK;
}

/* truncated_svd_factors (linalg.cpp:218-239).  Optional stats for logging. */
static void truncated_svd(const mat* m, size_t rank, mat* u_out, mat* v_out,
                          uint32_t* steps, uint64_t* iters, uint32_t* conv) {
  const size_t n = m->rows, mm = m->cols;
  mat u = mnew(n, rank), v = mnew(mm, rank);
  mat res = mcopy(m->a, n, mm);
  const double scale = fnorm(m);
  if (steps) { *steps = 0; *iters = 0; *conv = 0; }
  for (size_t k = 0; k < rank; ++k) {
    if (fnorm(&res) <= 1e-14 * scale) break;
    pair_t p = {0.0, NULL, NULL, 0, 0};
    top_pair(&res, 1000, 1e-13, &p);
    if (steps) { ++*steps; *iters += (uint64_t)p.iters; *conv += p.converged ? 1u : 0u; }
    const double root = sqrt(p.sigma);
    for (size_t i = 0; i < n; ++i) AT(u, i, k) = root * p.left[i];
    for (size_t j = 0; j < mm; ++j) AT(v, j, k) = root * p.right[j];
    for (size_t i = 0; i < n; ++i) {
      double* row = res.a + i * mm;
      const double ui = p.sigma * p.left[i];
      for (size_t j = 0; j < mm; ++j) row[j] -= ui * p.right[j];
    }
    free(p.left);
    free(p.right);
  }
  mfree(&res);
  *u_out = u;
  *v_out = v;
}
int nqo_truncated_svd(const double* a, uint32_t rows, uint32_t cols, uint32_t rank, double* u,
                      double* v) {
  mat m = {rows, cols, (double*)a}, uu, vv;
  truncated_svd(&m, rank, &uu, &vv, NULL, NULL, NULL);
  memcpy(u, uu.a, (size_t)rows * rank * sizeof(double));
  memcpy(v, vv.a, (size_t)cols * rank * sizeof(double));
  mfree(&uu);
  mfree(&vv);
  return NQB_OK;
}

static int cholesky_solve(const mat* a, const mat* b, mat* x_out) { /* linalg.cpp:140-176 */
  if (a->rows != a->cols || a->rows != b->rows) return NQB_E_DIMENSION_MISMATCH;
  if (!is_finite(b->a, b->rows * b->cols) || !is_finite(a->a, a->rows * a->cols))
    return NQB_E_NON_FINITE_INPUT;
  const size_t n = a->rows;
  double max_abs = 0.0, max_asym = 0.0, diag_sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    diag_sum += AT(*a, i, i);
    for (size_t j = 0; j < n; ++j) {
      const double x = fabs(AT(*a, i, j));
      if (x > max_abs) max_abs = x;
      if (j > i) {
        const double d = fabs(AT(*a, i, j) - AT(*a, j, i));
        if (d > max_asym) max_asym = d;
      }
    }
  }
  if (max_asym > 1e-9 * (max_abs > 1e-300 ? max_abs : 1e-300)) return NQB_E_NOT_SYMMETRIC;
  const double mean_diag = n > 0 ? diag_sum / (double)n : 0.0;
  static const double jitter[4] = {0.0, 1e-10, 1e-7, 1e-4};
  for (int t = 0; t < 4; ++t) {
    const double delta = jitter[t];
    mat l = mcopy(a->a, n, n);
    if (delta > 0.0) {
      const double add = delta * fabs(mean_diag);
      if (add == 0.0) { mfree(&l); continue; }
      for (size_t i = 0; i < n; ++i) AT(l, i, i) += add;
    }
    if (!try_cholesky(&l)) { mfree(&l); continue; }
    mat x = chol_backsolve(&l, b);
    mat ax = matmul(a, &x);
    mat res = msub(b, &ax);
    mat dx = chol_backsolve(&l, &res);
    mat x2 = madd(&x, &dx);
    mfree(&x); mfree(&ax); mfree(&res); mfree(&dx); mfree(&l);
    if (!is_finite(x2.a, x2.rows * x2.cols)) { mfree(&x2); continue; }
    *x_out = x2;
    return NQB_OK;
  }
  return NQB_E_NOT_POSITIVE_DEFINITE;
}
int nqo_cholesky_solve(const double* a, uint32_t n, const double* b, uint32_t nrhs, double* x) {
  mat am = {n, n, (double*)a}, bm = {n, nrhs, (double*)b}, xm;
  const int st = cholesky_solve(&am, &bm, &xm);
  if (st) return st;
  memcpy(x, xm.a, (size_t)n * nrhs * sizeof(double));
  mfree(&xm);
  return NQB_OK;
}

/* ------------------------------------------------------------------------ */
/* ADMM (admm.cpp:24-199)                                                    */
/* ------------------------------------------------------------------------ */
static int svid(const mat* p, mat* z_out) { /* admm.cpp:24-46 */
  const size_t n = p->rows * p->cols;
  if (!is_finite(p->a, n)) return NQB_E_NON_FINITE_INPUT;
  if (is_zero(p->a, n)) return NQB_E_ZERO_MATRIX;
  mat ab = mnew(p->rows, p->cols);
  for (size_t i = 0; i < n; ++i) ab.a[i] = fabs(p->a[i]);
  pair_t pr = {0.0, NULL, NULL, 0, 0};
  top_pair(&ab, 300, 1e-12, &pr);
  mfree(&ab);
  const double root = sqrt(pr.sigma);
  mat z = mnew(p->rows, p->cols);
  for (size_t i = 0; i < p->rows; ++i) {
    const double ai = root * pr.left[i];
    for (size_t j = 0; j < p->cols; ++j) {
      const double mag = ai * root * pr.right[j];
      AT(z, i, j) = AT(*p, i, j) < 0.0 ? -mag : mag;
    }
  }
  free(pr.left);
  free(pr.right);
  *z_out = z;
  return NQB_OK;
}
int nqo_svid(const double* p, uint32_t rows, uint32_t cols, double* z) {
  mat pm = {rows, cols, (double*)p}, zm;
  const int st = svid(&pm, &zm);
  if (st) return st;
  memcpy(z, zm.a, (size_t)rows * cols * sizeof(double));
  mfree(&zm);
  return NQB_OK;
}

static int factor_solve(const mat* target, const mat* fixed, const mat* z, const mat* l,
                        double rho, double ridge, mat* x_out) { /* admm.cpp:48-80 */
  const size_t r = fixed->cols;
  if (z->cols != r || l->cols != r) return NQB_E_DIMENSION_MISMATCH;
  if (z->rows != target->rows || l->rows != target->rows) return NQB_E_DIMENSION_MISMATCH;
  if (fixed->rows != target->cols) return NQB_E_DIMENSION_MISMATCH;
  mat a = matmul_at_b(fixed, fixed);
  for (size_t i = 0; i < r; ++i) AT(a, i, i) += rho + ridge;
  mat rhs = mnew(r, target->rows);
  for (size_t i = 0; i < target->rows; ++i) {
    const double* trow = target->a + i * target->cols;
    for (size_t k = 0; k < fixed->rows; ++k) {
      const double t = trow[k];
      if (t == 0.0) continue;
      const double* frow = fixed->a + k * r;
      for (size_t c = 0; c < r; ++c) AT(rhs, c, i) += t * frow[c];
    }
    const double* zr = z->a + i * r;
    const double* lr = l->a + i * r;
    for (size_t c = 0; c < r; ++c) AT(rhs, c, i) += rho * (zr[c] - lr[c]);
  }
  mat xt;
  const int st = cholesky_solve(&a, &rhs, &xt);
  mfree(&a);
  mfree(&rhs);
  if (st) return st;
  *x_out = transposed(&xt);
  mfree(&xt);
  return NQB_OK;
}
int nqo_factor_solve(const double* target, uint32_t rows, uint32_t cols, const double* fixed,
                     uint32_t rank, const double* z, const double* l, double rho,
                     double ridge, double* x) {
  mat tm = {rows, cols, (double*)target}, fm = {cols, rank, (double*)fixed};
  mat zm = {rows, rank, (double*)z}, lm = {rows, rank, (double*)l}, xm;
  const int st = factor_solve(&tm, &fm, &zm, &lm, rho, ridge, &xm);
  if (st) return st;
  memcpy(x, xm.a, (size_t)rows * rank * sizeof(double));
  mfree(&xm);
  return NQB_OK;
}

typedef struct { mat u, v, zu, zv, lu, lv; double rho; } state_t;

static double lagrangian(const state_t* s, const mat* target, double ridge) {
  mat vt = transposed(&s->v); /* admm.cpp:82-96 */
  mat approx = matmul(&s->u, &vt);
  mat d = msub(target, &approx);
  double value = 0.5 * sqnorm(&d);
  value += 0.5 * ridge * (sqnorm(&s->u) + sqnorm(&s->v));
  mat ru = msub(&s->u, &s->zu), rv = msub(&s->v, &s->zv);
  value += s->rho * mdot(&s->lu, &ru) + 0.5 * s->rho * sqnorm(&ru);
  value += s->rho * mdot(&s->lv, &rv) + 0.5 * s->rho * sqnorm(&rv);
  mfree(&vt); mfree(&approx); mfree(&d); mfree(&ru); mfree(&rv);
  return value;
}
int nqo_lagrangian(const double* u, const double* v, const double* zu, const double* zv,
                   const double* lu, const double* lv, uint32_t n, uint32_t m, uint32_t r,
                   double rho, const double* target, double ridge, double* out) {
  state_t s = {{n, r, (double*)u}, {m, r, (double*)v}, {n, r, (double*)zu},
               {m, r, (double*)zv}, {n, r, (double*)lu}, {m, r, (double*)lv}, rho};
  mat t = {n, m, (double*)target};
  *out = lagrangian(&s, &t, ridge);
  return NQB_OK;
}

static double rel_residual(const mat* x, const mat* z) { /* admm.cpp:104-108 */
  const double nx = fnorm(x);
  mat d = msub(x, z);
  const double r = fnorm(&d);
  mfree(&d);
  return r / (nx > 1e-300 ? nx : 1e-300);
}
static void rebalance(state_t* s) { /* admm.cpp:112-123 */
  const double nu = fnorm(&s->u), nv = fnorm(&s->v);
  if (nu <= 0.0 || nv <= 0.0) return;
  const double c = sqrt(nv / nu);
  mscale(&s->u, c); mscale(&s->zu, c); mscale(&s->lu, c);
  mscale(&s->v, 1.0 / c); mscale(&s->zv, 1.0 / c); mscale(&s->lv, 1.0 / c);
}

static int admm(const mat* target, const nqb_admm_config* cfg, mat* cu, mat* cv,
                double* trace, nqb_admm_result* res) { /* admm.cpp:127-199 */
  const size_t n = target->rows, m = target->cols;
  if (is_zero(target->a, n * m)) return NQB_E_ZERO_MATRIX;
  if (!is_finite(target->a, n * m)) return NQB_E_NON_FINITE_INPUT;
  if (cfg->rank == 0) return NQB_E_INVALID_RANK;
  if (cfg->rank > (n < m ? n : m)) return NQB_E_RANK_TOO_LARGE;
  if (cfg->max_iters < 1) return NQB_E_VALIDATION;
  memset(res, 0, sizeof(*res));
  double rho_start = cfg->rho_start, rho_end = cfg->rho_end;
  if (rho_start <= 0.0 && rho_end <= 0.0) {
    double spectral = spectral_norm(target, 200);
    if (spectral < 1e-12) spectral = 1e-12;
    res->sigma_max = spectral;
    rho_start = 0.1 * spectral;
    rho_end = 10.0 * spectral;
  } else if (rho_start <= 0.0 || rho_end < rho_start) {
    return NQB_E_VALIDATION;
  }
  state_t s;
  truncated_svd(target, cfg->rank, &s.u, &s.v, &res->svd_steps, &res->svd_power_iters,
                &res->svd_converged_steps);
  int st = svid(&s.u, &s.zu);
  if (st) return st;
  st = svid(&s.v, &s.zv);
  if (st) return st;
  s.lu = mnew(s.u.rows, s.u.cols);
  s.lv = mnew(s.v.rows, s.v.cols);
  s.rho = rho_start;
  uint32_t tl = 0;
  if (trace) trace[tl++] = lagrangian(&s, target, cfg->ridge);
  mat wt = transposed(target);
  const int denom = cfg->max_iters - 1 > 1 ? cfg->max_iters - 1 : 1;
  int converged = 0;
  uint32_t iteration = 0;
  double primal = 0.0;
  for (int k = 0; k < cfg->max_iters; ++k) {
    const double r1 = rel_residual(&s.u, &s.zu), r2 = rel_residual(&s.v, &s.zv);
    primal = r1 > r2 ? r1 : r2;
    if (primal < cfg->tol) { converged = 1; break; }
    const double rho = rho_start + (rho_end - rho_start) * ((double)k / denom);
    if (rho != s.rho) {
      const double rescale = s.rho / rho;
      mscale(&s.lu, rescale);
      mscale(&s.lv, rescale);
      s.rho = rho;
    }
    rebalance(&s);
    mat nu, nv, pu, pv, du, dv;
    if ((st = factor_solve(target, &s.v, &s.zu, &s.lu, s.rho, cfg->ridge, &nu))) return st;
    mfree(&s.u); s.u = nu;
    if ((st = factor_solve(&wt, &s.u, &s.zv, &s.lv, s.rho, cfg->ridge, &nv))) return st;
    mfree(&s.v); s.v = nv;
    pu = madd(&s.u, &s.lu);
    pv = madd(&s.v, &s.lv);
    mfree(&s.zu); mfree(&s.zv);
    if ((st = svid(&pu, &s.zu))) return st;
    if ((st = svid(&pv, &s.zv))) return st;
    mfree(&pu); mfree(&pv);
    du = msub(&s.u, &s.zu);
    dv = msub(&s.v, &s.zv);
    pu = madd(&s.lu, &du);
    pv = madd(&s.lv, &dv);
    mfree(&du); mfree(&dv); mfree(&s.lu); mfree(&s.lv);
    s.lu = pu;
    s.lv = pv;
    iteration = (uint32_t)k + 1;
    if (trace) trace[tl++] = lagrangian(&s, target, cfg->ridge);
  }
  if (!converged) {
    const double r1 = rel_residual(&s.u, &s.zu), r2 = rel_residual(&s.v, &s.zv);
    primal = r1 > r2 ? r1 : r2;
    converged = primal < cfg->tol;
  }
  mfree(&wt);
  *cu = madd(&s.u, &s.lu);
  *cv = madd(&s.v, &s.lv);
  res->iteration = iteration;
  res->converged = converged;
  res->primal_residual = primal;
  res->rho = s.rho;
  res->trace_len = tl;
  mfree(&s.u); mfree(&s.v); mfree(&s.zu); mfree(&s.zv); mfree(&s.lu); mfree(&s.lv);
  return NQB_OK;
}
int nqo_admm_factorize(const double* w, uint32_t n, uint32_t m, const nqb_admm_config* cfg,
                       double* cu, double* cv, double* trace, nqb_admm_result* res) {
  mat t = {n, m, (double*)w}, a, b;
  const int st = admm(&t, cfg, &a, &b, trace, res);
  if (st) return st;
  memcpy(cu, a.a, (size_t)n * cfg->rank * sizeof(double));
  memcpy(cv, b.a, (size_t)m * cfg->rank * sizeof(double));
  mfree(&a);
  mfree(&b);
  return NQB_OK;
}

/* ------------------------------------------------------------------------ */
/* Balance (balance.cpp:23-65, precondition.cpp:143-153)                     */
/* ------------------------------------------------------------------------ */
static void unprecondition(mat* f, const double* diag) {
  if (!diag) return;
  for (size_t i = 0; i < f->rows; ++i) {
    const double inv = 1.0 / diag[i];
    for (size_t j = 0; j < f->cols; ++j) AT(*f, i, j) *= inv;
  }
}
static void row_mean_abs(const mat* m, double floor, double* out) {
  for (size_t i = 0; i < m->rows; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < m->cols; ++j) s += fabs(AT(*m, i, j));
    const double v = s / (double)m->cols;
    out[i] = (v < floor) ? floor : v; /* std::max(v, floor) */
  }
}
static double balance(mat* lu, mat* lv, const double* diag_out, const double* diag_in,
                      double floor, double* s1, double* s2) {
  unprecondition(lu, diag_out);
  unprecondition(lv, diag_in);
  const double nu = fnorm(lu), nv = fnorm(lv);
  const double eta = (nu == 0.0 || nv == 0.0) ? 1.0 : sqrt(nv / nu);
  mscale(lu, eta);
  mscale(lv, 1.0 / eta);
  row_mean_abs(lu, floor, s1);
  row_mean_abs(lv, floor, s2);
  return eta;
}
int nqo_balance(const double* pu, const double* pv, uint32_t n, uint32_t m, uint32_t r,
                const double* diag_out, const double* diag_in, double floor, double* lu,
                double* lv, double* s1, double* s2, double* eta) {
  mat a = mcopy(pu, n, r), b = mcopy(pv, m, r);
  *eta = balance(&a, &b, diag_out, diag_in, floor, s1, s2);
  memcpy(lu, a.a, (size_t)n * r * sizeof(double));
  memcpy(lv, b.a, (size_t)m * r * sizeof(double));
  mfree(&a);
  mfree(&b);
  return NQB_OK;
}

/* Per-matrix pipeline step (pipeline.cpp:95-110, :150-153). */
int nqo_factorize_layer(const double* w, uint32_t n, uint32_t m, const nqb_admm_config* cfg,
                        double floor, uint32_t* u_words, uint32_t* v_words, double* s1,
                        double* s2, double* rel_err, double* trace, nqb_admm_result* res) {
  mat t = {n, m, (double*)w}, cu, cv;
  int st = admm(&t, cfg, &cu, &cv, trace, res);
  if (st) return st;
  balance(&cu, &cv, NULL, NULL, floor, s1, s2);
  if ((st = pack_latent(&cu, u_words)) || (st = pack_latent(&cv, v_words))) return st;
  mat rec = mnew(n, m);
  reconstruct(n, m, cfg->rank, u_words, v_words, s1, s2, rec.a);
  *rel_err = rel_fro_error(&t, &rec);
  mfree(&rec);
  mfree(&cu);
  mfree(&cv);
  return NQB_OK;
}

int nqo_layer_rel_error(uint32_t n, uint32_t m, uint32_t r, const uint32_t* u,
                        const uint32_t* v, const double* s1, const double* s2,
                        const double* w, double* out) {
  mat t = {n, m, (double*)w}, rec = mnew(n, m);
  reconstruct(n, m, r, u, v, s1, s2, rec.a);
  *out = rel_fro_error(&t, &rec);
  mfree(&rec);
  return NQB_OK;
}

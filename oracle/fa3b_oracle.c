/* TEST INFRASTRUCTURE ONLY — CPU oracle for the fa3b hot path.
 *
 * Plain-C restatement of the reference (flashlab proj/core) attention
 * algorithms; see fa3b_oracle.h for the contract. Compiled with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:16-18) and with
 * the same per-element operation order, so the FP64 paths reproduce the
 * reference bit for bit (checked in tests/test_oracle.py against oracle/_ref).
 */
#define _GNU_SOURCE
#include "fa3b_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static _Thread_local const char* g_err = "";
const char* fa3b_oracle_last_error(void) { return g_err; }
static int fail(const char* msg) {
  g_err = msg;
  return -1;
}

/* ------------------------------------------------------------------ rng.cpp */
static const uint64_t kGamma = 0x9E3779B97F4A7C15ull;

static uint64_t mix64(uint64_t z) { /* rng.cpp:15-19 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t orc_substream(uint64_t seed, uint64_t salt) { /* rng.cpp:21-23 */
  return mix64(seed ^ mix64(salt + kGamma));
}
uint64_t orc_word(uint64_t seed, uint64_t c) { return mix64(seed + (c + 1) * kGamma); }
static double uniform(uint64_t seed, uint64_t c) { /* rng.cpp:29-31 */
  return (double)(orc_word(seed, c) >> 11) * 0x1.0p-53;
}
static double uniform_pos(uint64_t seed, uint64_t c) { /* rng.cpp:33-35 */
  return (double)((orc_word(seed, c) >> 11) + 1) * 0x1.0p-53;
}
double orc_gaussian(uint64_t seed, uint64_t c) { /* rng.cpp:37-41, Box-Muller */
  const double u1 = uniform_pos(seed, 2 * c);
  const double u2 = uniform(seed, 2 * c + 1);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}
void orc_sample_gaussian(size_t rows, size_t cols, uint64_t seed, double* out) {
  for (size_t i = 0; i < rows * cols; ++i) out[i] = orc_gaussian(seed, i); /* rng.cpp:43-48 */
}
int orc_sample_outlier(size_t rows, size_t cols, uint64_t seed, double p, double* out) {
  /* rng.cpp:50-71: N(0,1) + 10 N(0,1) Bern(p), five words per entry */
  if (p < 0.0 || p > 1.0) return fail("sample_outlier_matrix: probability out of range");
  for (size_t e = 0; e < rows * cols; ++e) {
    const uint64_t base = 5 * e;
    const double u1 = uniform_pos(seed, base);
    const double u2 = uniform(seed, base + 1);
    double v = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
    if (uniform(seed, base + 2) < p) {
      const double u3 = uniform_pos(seed, base + 3);
      const double u4 = uniform(seed, base + 4);
      v += 10.0 * (sqrt(-2.0 * log(u3)) * cos(2.0 * M_PI * u4));
    }
    out[e] = v;
  }
  return 0;
}
void orc_sign_vector(size_t n, uint64_t seed, double* out) { /* rng.cpp:73-78 */
  for (size_t i = 0; i < n; ++i) out[i] = (orc_word(seed, i) & 1ull) ? 1.0 : -1.0;
}

/* -------------------------------------------------------------- formats.cpp */
typedef struct {
  int ebits, mbits;
  double max_finite;
} Fmt;
static const Fmt kFmts[5] = {
    {11, 52, DBL_MAX}, {8, 23, 0x1.FFFFFEp127}, {5, 10, 65504.0}, {8, 7, 0x1.FEp127},
    {4, 3, 448.0}, /* e4m3 OCP FN: S.1111.111 is NaN (formats.cpp:18-25) */
};
double orc_round_to(double x, int fmt, int overflow_infinite) { /* formats.cpp:45-61 */
  if (fmt == ORC_FP64 || isnan(x) || x == 0.0 || isinf(x)) return x;
  const Fmt f = kFmts[fmt];
  const int bias = (1 << (f.ebits - 1)) - 1;
  const int min_normal_exp = 1 - bias;
  const double ax = fabs(x);
  int e = ilogb(ax);
  if (e < min_normal_exp) e = min_normal_exp;
  const double q = ldexp(1.0, e - f.mbits);
  double r = nearbyint(ax / q) * q; /* ties to even */
  if (r > f.max_finite) r = overflow_infinite ? INFINITY : f.max_finite;
  return copysign(r, x);
}
static double to_f32(double x) { return (double)(float)x; }
void orc_round_array(const double* in, size_t n, int fmt, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_round_to(in[i], fmt, 0);
}

/* --------------------------------------------------------------- matrix.cpp */
/* c[m x n] = a[m x k] * b^T where b is [n x k] (transpose_b) or b[k x n];
 * FP64, k ascending per entry (matrix.cpp:27-42, matrix.hpp:67-79). */
static void matmul(const double* a, size_t m, size_t k, const double* b, size_t n,
                   int transpose_b, double* c) {
  memset(c, 0, sizeof(double) * m * n);
  for (size_t i = 0; i < m; ++i)
    for (size_t p = 0; p < k; ++p) {
      const double av = a[i * k + p];
      for (size_t j = 0; j < n; ++j)
        c[i * n + j] += av * (transpose_b ? b[j * k + p] : b[p * n + j]);
    }
}
/* float accumulator, code-level products (quantize.cpp:80-135) */
static void matmul_f32(const double* a, size_t m, size_t k, const double* b, size_t n,
                       int transpose_b, float* c) {
  memset(c, 0, sizeof(float) * m * n);
  for (size_t i = 0; i < m; ++i)
    for (size_t p = 0; p < k; ++p) {
      const float av = (float)a[i * k + p];
      for (size_t j = 0; j < n; ++j)
        c[i * n + j] += av * (float)(transpose_b ? b[j * k + p] : b[p * n + j]);
    }
}

/* ------------------------------------------------------------- hadamard.cpp */
int orc_fwht(double* v, size_t n) { /* hadamard.cpp:11-27 */
  if (n == 0 || (n & (n - 1))) return fail("fwht: length must be a power of two");
  for (size_t len = 1; len < n; len <<= 1)
    for (size_t i = 0; i < n; i += len << 1)
      for (size_t j = i; j < i + len; ++j) {
        const double a = v[j], b = v[j + len];
        v[j] = a + b;
        v[j + len] = a - b;
      }
  const double norm = 1.0 / sqrt((double)n);
  for (size_t i = 0; i < n; ++i) v[i] *= norm;
  return 0;
}
int orc_preprocess_incoherent(const double* q, const double* k, size_t n, size_t d,
                              uint64_t seed, double* qo, double* ko) {
  /* fp8_attention.cpp:33-42 -> random_dh_transform (hadamard.cpp:60-64), apply
   * = sign flip then normalized FWHT (hadamard.cpp:29-33) on every row */
  if (d == 0 || (d & (d - 1))) return fail("random_dh_transform: dim must be a power of two");
  double* s = malloc(sizeof(double) * d);
  orc_sign_vector(d, seed, s);
  for (int which = 0; which < 2; ++which) {
    const double* src = which ? k : q;
    double* dst = which ? ko : qo;
    for (size_t r = 0; r < n; ++r) {
      for (size_t j = 0; j < d; ++j) dst[r * d + j] = src[r * d + j] * s[j];
      orc_fwht(dst + r * d, d);
    }
  }
  free(s);
  return 0;
}

/* ------------------------------------------------------------- quantize.cpp */
static int encode_block(const double* m, size_t r0, size_t r1, size_t cols, int ov,
                        double* codes, double* scale_out) {
  double amax = 0.0; /* quantize.cpp:10-21 */
  for (size_t i = r0 * cols; i < r1 * cols; ++i) {
    const double a = fabs(m[i]);
    if (!isfinite(a)) return fail("quantize: non-finite input entry");
    if (a > amax) amax = a;
  }
  const double scale = amax == 0.0 ? 1.0 : amax / 448.0; /* quantize.cpp:40,55 */
  const double inv = 1.0 / scale;                         /* quantize.cpp:25 */
  for (size_t i = r0 * cols; i < r1 * cols; ++i) codes[i] = orc_round_to(m[i] * inv, ORC_E4M3, ov);
  *scale_out = scale;
  return 0;
}
int orc_quantize(const double* m, size_t rows, size_t cols, size_t block_rows,
                 int overflow_infinite, double* codes, double* scales) {
  if (rows == 0 || cols == 0)
    return fail(block_rows ? "quantize_per_block: empty matrix" : "quantize_per_tensor: empty matrix");
  if (block_rows == 0) return encode_block(m, 0, rows, cols, overflow_infinite, codes, scales);
  for (size_t r0 = 0, b = 0; r0 < rows; r0 += block_rows, ++b) {
    const size_t r1 = r0 + block_rows < rows ? r0 + block_rows : rows;
    if (encode_block(m, r0, r1, cols, overflow_infinite, codes, scales + b)) return -1;
  }
  return 0;
}

/* --------------------------------------------------------- attention_ref.cpp */
static int validate(size_t n, size_t d, double alpha) { /* attention_ref.cpp:20-29 */
  if (n == 0 || d == 0) return fail("attention: empty inputs");
  if (!isfinite(alpha) || alpha == 0.0) return fail("attention: alpha must be finite and nonzero");
  return 0;
}
static int check_tile(size_t br, size_t bc) { /* flash_fwd.cpp:127-129 */
  if (br == 0 || bc == 0) return fail("TileConfig: block sizes must be positive");
  return 0;
}

int orc_reference_attention(const double* q, const double* k, const double* v, size_t n,
                            size_t d, double alpha, int causal, double* o, double* lse) {
  /* attention_ref.cpp:36-76,116-128 with block_rows = 128 */
  if (validate(n, d, alpha)) return -1;
  const size_t br = 128;
  double* s = malloc(sizeof(double) * br * n);
  double* ob = malloc(sizeof(double) * br * d);
  for (size_t r0 = 0; r0 < n; r0 += br) {
    const size_t nr = r0 + br < n ? br : n - r0;
    matmul(q + r0 * d, nr, d, k, n, 1, s);
    for (size_t i = 0; i < nr; ++i) {
      double* row = s + i * n;
      for (size_t j = 0; j < n; ++j) row[j] *= alpha;
      if (causal)
        for (size_t j = r0 + i + 1; j < n; ++j) row[j] = -INFINITY;
    }
    for (size_t i = 0; i < nr; ++i) {
      double* row = s + i * n;
      double m = -INFINITY;
      for (size_t j = 0; j < n; ++j)
        if (row[j] > m) m = row[j];
      if (m == -INFINITY) {
        for (size_t j = 0; j < n; ++j) row[j] = 0.0;
        lse[r0 + i] = -INFINITY;
        continue;
      }
      double ell = 0.0;
      for (size_t j = 0; j < n; ++j) {
        const double e = exp(row[j] - m);
        row[j] = e;
        ell += e;
      }
      const double inv = 1.0 / ell;
      for (size_t j = 0; j < n; ++j) row[j] *= inv;
      lse[r0 + i] = m + log(ell);
    }
    matmul(s, nr, n, v, d, 0, ob);
    memcpy(o + r0 * d, ob, sizeof(double) * nr * d);
  }
  free(s);
  free(ob);
  return 0;
}

/* ------------------------------------------------------------ flash_fwd.cpp */
int orc_flash_fwd(const double* q, const double* k, const double* v, size_t n, size_t d,
                  double alpha, int causal, size_t br, size_t bc, double* o, double* lse,
                  uint64_t* visited, uint64_t* skipped) {
  if (validate(n, d, alpha) || check_tile(br, bc)) return -1;
  double* s = malloc(sizeof(double) * br * bc);
  double* g = malloc(sizeof(double) * br * d);
  double* oacc = malloc(sizeof(double) * br * d);
  double* m = malloc(sizeof(double) * br);
  double* ell = malloc(sizeof(double) * br);
  uint64_t nvis = 0, nskip = 0;
  for (size_t r0 = 0; r0 < n; r0 += br) {
    const size_t nr = r0 + br < n ? br : n - r0;
    for (size_t i = 0; i < nr; ++i) m[i] = -INFINITY, ell[i] = 0.0;
    memset(oacc, 0, sizeof(double) * nr * d);
    for (size_t c0 = 0; c0 < n; c0 += bc) {
      const size_t nc = c0 + bc < n ? bc : n - c0;
      if (causal && c0 > r0 + nr - 1) { /* active_col_blocks, flash_fwd.cpp:110-124 */
        ++nskip;
        continue;
      }
      ++nvis;
      /* score_block (flash_fwd.cpp:57-71) */
      matmul(q + r0 * d, nr, d, k + c0 * d, nc, 1, s);
      for (size_t i = 0; i < nr; ++i) {
        double* row = s + i * nc;
        for (size_t j = 0; j < nc; ++j) row[j] *= alpha;
        if (causal)
          for (size_t j = 0; j < nc; ++j)
            if (c0 + j > r0 + i) row[j] = -INFINITY;
      }
      /* online_softmax_step (flash_fwd.cpp:18-48) */
      for (size_t i = 0; i < nr; ++i) {
        double* row = s + i * nc;
        double m_new = m[i];
        for (size_t j = 0; j < nc; ++j)
          if (row[j] > m_new) m_new = row[j];
        double r;
        if (m_new == -INFINITY) {
          r = 0.0;
          for (size_t j = 0; j < nc; ++j) row[j] = 0.0;
        } else {
          r = exp(m[i] - m_new);
          double bsum = 0.0;
          for (size_t j = 0; j < nc; ++j) {
            const double e = exp(row[j] - m_new);
            row[j] = e;
            bsum += e;
          }
          ell[i] = r * ell[i] + bsum;
          m[i] = m_new;
        }
        /* accumulate_output scale step (flash_fwd.cpp:78-82) */
        for (size_t j = 0; j < d; ++j) oacc[i * d + j] *= r;
      }
      matmul(s, nr, nc, v + c0 * d, d, 0, g); /* flash_fwd.cpp:83-89 */
      for (size_t i = 0; i < nr * d; ++i) oacc[i] += g[i];
    }
    for (size_t i = 0; i < nr; ++i) { /* epilogue, flash_fwd.cpp:92-106 */
      if (ell[i] > 0.0) {
        const double inv = 1.0 / ell[i];
        for (size_t j = 0; j < d; ++j) o[(r0 + i) * d + j] = oacc[i * d + j] * inv;
        lse[r0 + i] = m[i] + log(ell[i]);
      } else {
        for (size_t j = 0; j < d; ++j) o[(r0 + i) * d + j] = 0.0;
        lse[r0 + i] = -INFINITY;
      }
    }
  }
  if (visited) *visited = nvis;
  if (skipped) *skipped = nskip;
  free(s), free(g), free(oacc), free(m), free(ell);
  return 0;
}

/* ------------------------------------------------------------ flash_bwd.cpp */
int orc_bwd_preprocess(const double* dO, const double* o, size_t n, size_t d, double* out) {
  for (size_t i = 0; i < n; ++i) { /* flash_bwd.cpp:29-41 */
    double acc = 0.0;
    for (size_t j = 0; j < d; ++j) acc += dO[i * d + j] * o[i * d + j];
    out[i] = acc;
  }
  return 0;
}

/* Shared KV-outer / Q-inner loop (flash_bwd.cpp:58-125). fmt = ORC_FP64
 * reproduces the reference exactly; a 16-bit fmt rounds inputs, P and dS to
 * fmt and accumulates the GEMMs in fp32 (tensor-core semantics). */
static int bwd_impl(const double* q_, const double* k_, const double* v_, const double* dO_,
                    const double* o_, const double* lse, size_t n, size_t d, double alpha,
                    int causal, size_t br, size_t bc, int fmt, double* dq, double* dk,
                    double* dv) {
  if (validate(n, d, alpha) || check_tile(br, bc)) return -1;
  const int lp = fmt != ORC_FP64;
  const double *q = q_, *k = k_, *v = v_, *dO = dO_, *o = o_;
  double* rounded[5] = {0};
  if (lp) {
    const double* src[5] = {q_, k_, v_, dO_, o_};
    for (int t = 0; t < 5; ++t) {
      rounded[t] = malloc(sizeof(double) * n * d);
      for (size_t i = 0; i < n * d; ++i) rounded[t][i] = orc_round_to(src[t][i], fmt, 0);
    }
    q = rounded[0], k = rounded[1], v = rounded[2], dO = rounded[3], o = rounded[4];
  }
  double* D = malloc(sizeof(double) * n);
  orc_bwd_preprocess(dO, o, n, d, D);
  if (lp)
    for (size_t i = 0; i < n; ++i) D[i] = to_f32(D[i]);
  double* p = malloc(sizeof(double) * br * bc);
  double* pT = malloc(sizeof(double) * bc * br);
  double* dp = malloc(sizeof(double) * br * bc);
  double* ds = malloc(sizeof(double) * br * bc);
  double* dsT = malloc(sizeof(double) * bc * br);
  double* tmp = malloc(sizeof(double) * (br > bc ? br : bc) * d);
  double* dkj = malloc(sizeof(double) * bc * d);
  double* dvj = malloc(sizeof(double) * bc * d);
  float* f32 = malloc(sizeof(float) * (br + bc) * (d + br + bc));
  memset(dq, 0, sizeof(double) * n * d);
#define GEMM(a, m_, k__, b, n_, tb, out)                                      \
  do {                                                                        \
    if (lp) {                                                                 \
      matmul_f32(a, m_, k__, b, n_, tb, f32);                                 \
      for (size_t z_ = 0; z_ < (size_t)(m_) * (n_); ++z_) out[z_] = f32[z_]; \
    } else {                                                                  \
      matmul(a, m_, k__, b, n_, tb, out);                                     \
    }                                                                         \
  } while (0)
  for (size_t c0 = 0; c0 < n; c0 += bc) {
    const size_t nc = c0 + bc < n ? bc : n - c0;
    memset(dkj, 0, sizeof(double) * nc * d);
    memset(dvj, 0, sizeof(double) * nc * d);
    for (size_t r0 = 0; r0 < n; r0 += br) {
      const size_t nr = r0 + br < n ? br : n - r0;
      if (causal && r0 + nr - 1 < c0) continue;
      GEMM(q + r0 * d, nr, d, k + c0 * d, nc, 1, p);
      for (size_t i = 0; i < nr; ++i) {
        double* row = p + i * nc;
        for (size_t j = 0; j < nc; ++j) row[j] *= alpha;
        if (causal)
          for (size_t j = 0; j < nc; ++j)
            if (c0 + j > r0 + i) row[j] = -INFINITY;
        const double l = lse[r0 + i];
        if (l == -INFINITY) {
          for (size_t j = 0; j < nc; ++j) row[j] = 0.0;
        } else {
          for (size_t j = 0; j < nc; ++j) row[j] = exp(row[j] - l);
        }
      }
      /* dV_j += P^T dO_i (the GEMM operand P is fmt-rounded on the device) */
      for (size_t i = 0; i < nr; ++i)
        for (size_t j = 0; j < nc; ++j) pT[j * nr + i] = lp ? orc_round_to(p[i * nc + j], fmt, 0) : p[i * nc + j];
      GEMM(pT, nc, nr, dO + r0 * d, d, 0, tmp);
      for (size_t i = 0; i < nc * d; ++i) dvj[i] += tmp[i];
      GEMM(dO + r0 * d, nr, d, v + c0 * d, nc, 1, dp);
      for (size_t i = 0; i < nr; ++i)
        for (size_t j = 0; j < nc; ++j) {
          double x = p[i * nc + j] * (dp[i * nc + j] - D[r0 + i]);
          if (lp) x = orc_round_to(x, fmt, 0);
          ds[i * nc + j] = x;
          dsT[j * nr + i] = x;
        }
      GEMM(ds, nr, nc, k + c0 * d, d, 0, tmp);
      for (size_t i = 0; i < nr * d; ++i) dq[r0 * d + i] += tmp[i];
      GEMM(dsT, nc, nr, q + r0 * d, d, 0, tmp);
      for (size_t i = 0; i < nc * d; ++i) dkj[i] += tmp[i];
    }
    for (size_t i = 0; i < nc * d; ++i) { /* alpha folds in once (flash_bwd.cpp:111-119) */
      dk[c0 * d + i] = alpha * dkj[i];
      dv[c0 * d + i] = dvj[i];
    }
  }
#undef GEMM
  for (size_t i = 0; i < n * d; ++i) dq[i] *= alpha; /* flash_bwd.cpp:121-124 */
  for (int t = 0; t < 5; ++t) free(rounded[t]);
  free(D), free(p), free(pT), free(dp), free(ds), free(dsT), free(tmp), free(dkj), free(dvj),
      free(f32);
  return 0;
}
int orc_flash_bwd(const double* q, const double* k, const double* v, const double* dO,
                  const double* o, const double* lse, size_t n, size_t d, double alpha,
                  int causal, size_t br, size_t bc, double* dq, double* dk, double* dv) {
  return bwd_impl(q, k, v, dO, o, lse, n, d, alpha, causal, br, bc, ORC_FP64, dq, dk, dv);
}
int orc_lowprec_flash_bwd(const double* q, const double* k, const double* v,
                          const double* dO, const double* o, const double* lse, size_t n,
                          size_t d, double alpha, int causal, size_t br, size_t bc, int fmt,
                          double* dq, double* dk, double* dv) {
  return bwd_impl(q, k, v, dO, o, lse, n, d, alpha, causal, br, bc, fmt, dq, dk, dv);
}

/* -------------------------------------------------------------- lowprec.cpp */
int orc_lowprec_flash_fwd(const double* q_, const double* k_, const double* v_, size_t n,
                          size_t d, double alpha, int causal, size_t br, size_t bc, int fmt,
                          double* o, double* lse) {
  /* lowprec.cpp:166-240 with fp16 replaced by fmt */
  if (validate(n, d, alpha) || check_tile(br, bc)) return -1;
  double* q = malloc(sizeof(double) * n * d);
  double* k = malloc(sizeof(double) * n * d);
  double* v = malloc(sizeof(double) * n * d);
  for (size_t i = 0; i < n * d; ++i) {
    q[i] = orc_round_to(q_[i], fmt, 0);
    k[i] = orc_round_to(k_[i], fmt, 0);
    v[i] = orc_round_to(v_[i], fmt, 0);
  }
  float* sf = malloc(sizeof(float) * br * (bc > d ? bc : d));
  double* s = malloc(sizeof(double) * br * bc);
  double* oacc = malloc(sizeof(double) * br * d);
  double* m = malloc(sizeof(double) * br);
  double* ell = malloc(sizeof(double) * br);
  double* resc = malloc(sizeof(double) * br);
  for (size_t r0 = 0; r0 < n; r0 += br) {
    const size_t nr = r0 + br < n ? br : n - r0;
    for (size_t i = 0; i < nr; ++i) m[i] = -INFINITY, ell[i] = 0.0;
    memset(oacc, 0, sizeof(double) * nr * d);
    for (size_t c0 = 0; c0 < n; c0 += bc) {
      const size_t nc = c0 + bc < n ? bc : n - c0;
      if (causal && c0 > r0 + nr - 1) continue;
      matmul_f32(q + r0 * d, nr, d, k + c0 * d, nc, 1, sf);
      for (size_t i = 0; i < nr * nc; ++i) s[i] = to_f32((double)sf[i] * alpha);
      for (size_t i = 0; i < nr; ++i) {
        double* row = s + i * nc;
        resc[i] = 0.0;
        if (causal)
          for (size_t j = 0; j < nc; ++j)
            if (c0 + j > r0 + i) row[j] = -INFINITY;
        double m_new = m[i];
        for (size_t j = 0; j < nc; ++j) m_new = row[j] > m_new ? row[j] : m_new;
        if (m_new == -INFINITY) {
          for (size_t j = 0; j < nc; ++j) row[j] = 0.0;
          continue;
        }
        const double r = to_f32(exp(m[i] - m_new));
        double bsum = 0.0;
        for (size_t j = 0; j < nc; ++j) {
          const double e = to_f32(exp(row[j] - m_new));
          bsum = to_f32(bsum + e);
          row[j] = orc_round_to(e, fmt, 0);
        }
        ell[i] = to_f32(to_f32(r * ell[i]) + bsum);
        m[i] = m_new;
        resc[i] = r;
      }
      matmul_f32(s, nr, nc, v + c0 * d, d, 0, sf);
      for (size_t i = 0; i < nr; ++i)
        for (size_t j = 0; j < d; ++j)
          oacc[i * d + j] = to_f32(to_f32(oacc[i * d + j] * resc[i]) + (double)sf[i * d + j]);
    }
    for (size_t i = 0; i < nr; ++i) {
      if (ell[i] > 0.0) {
        for (size_t j = 0; j < d; ++j)
          o[(r0 + i) * d + j] = orc_round_to(oacc[i * d + j] / ell[i], fmt, 0);
        lse[r0 + i] = m[i] + log(ell[i]);
      } else {
        for (size_t j = 0; j < d; ++j) o[(r0 + i) * d + j] = 0.0;
        lse[r0 + i] = -INFINITY;
      }
    }
  }
  free(q), free(k), free(v), free(sf), free(s), free(oacc), free(m), free(ell), free(resc);
  return 0;
}

/* -------------------------------------------------------- fp8_attention.cpp */
int orc_fp8_flash_fwd(const double* q_, const double* k_, const double* v, size_t n, size_t d,
                      double alpha, int causal, int per_block, int incoherent, uint64_t seed,
                      size_t br, size_t bc, double* o, double* lse) {
  if (validate(n, d, alpha)) return -1;
  if (br == 0 || bc == 0) return fail("fp8_flash_fwd: tile sizes must be positive");
  double* q = malloc(sizeof(double) * n * d);
  double* k = malloc(sizeof(double) * n * d);
  if (incoherent) { /* fp8_attention.cpp:88-93 */
    if (orc_preprocess_incoherent(q_, k_, n, d, seed, q, k)) {
      free(q), free(k);
      return -1;
    }
  } else {
    memcpy(q, q_, sizeof(double) * n * d);
    memcpy(k, k_, sizeof(double) * n * d);
  }
  /* fp8_attention.cpp:94-96: Q per B_r rows, K and V per B_c rows */
  const size_t nbq = per_block ? (n + br - 1) / br : 1, nbk = per_block ? (n + bc - 1) / bc : 1;
  double* qc = malloc(sizeof(double) * n * d);
  double* kc = malloc(sizeof(double) * n * d);
  double* vc = malloc(sizeof(double) * n * d);
  double* sq = malloc(sizeof(double) * nbq);
  double* sk = malloc(sizeof(double) * nbk);
  double* sv = malloc(sizeof(double) * nbk);
  int rc = orc_quantize(q, n, d, per_block ? br : 0, 0, qc, sq);
  rc = rc ? rc : orc_quantize(k, n, d, per_block ? bc : 0, 0, kc, sk);
  rc = rc ? rc : orc_quantize(v, n, d, per_block ? bc : 0, 0, vc, sv);
  float* acc = malloc(sizeof(float) * br * (bc > d ? bc : d));
  double* s = malloc(sizeof(double) * br * bc);
  double* pc = malloc(sizeof(double) * br * bc);
  double* oacc = malloc(sizeof(double) * br * d);
  double* m = malloc(sizeof(double) * br);
  double* ell = malloc(sizeof(double) * br);
  double* resc = malloc(sizeof(double) * br);
  for (size_t r0 = 0; rc == 0 && r0 < n; r0 += br) {
    const size_t nr = r0 + br < n ? br : n - r0;
    const double sqv = per_block ? sq[r0 / br] : sq[0];
    for (size_t i = 0; i < nr; ++i) m[i] = -INFINITY, ell[i] = 0.0;
    memset(oacc, 0, sizeof(double) * nr * d);
    for (size_t c0 = 0; c0 < n; c0 += bc) {
      const size_t nc = c0 + bc < n ? bc : n - c0;
      if (causal && c0 > r0 + nr - 1) continue;
      const double skv = per_block ? sk[c0 / bc] : sk[0];
      const double svv = per_block ? sv[c0 / bc] : sv[0];
      /* S on codes; emulated_matmul applies unit scales (x 1.0) then the
       * kernel's descale (fp8_attention.cpp:113-124) */
      matmul_f32(qc + r0 * d, nr, d, kc + c0 * d, nc, 1, acc);
      const double descale = alpha * sqv * skv;
      for (size_t i = 0; i < nr; ++i)
        for (size_t j = 0; j < nc; ++j) {
          double x = to_f32(((double)acc[i * nc + j] * (1.0 * 1.0)) * descale);
          if (causal && c0 + j > r0 + i) x = -INFINITY;
          s[i * nc + j] = x;
        }
      /* online_softmax_step in FP64 (flash_fwd.cpp:18-48) */
      double pamax = 0.0;
      for (size_t i = 0; i < nr; ++i) {
        double* row = s + i * nc;
        double m_new = m[i];
        for (size_t j = 0; j < nc; ++j)
          if (row[j] > m_new) m_new = row[j];
        if (m_new == -INFINITY) {
          resc[i] = 0.0;
          for (size_t j = 0; j < nc; ++j) row[j] = 0.0;
          continue;
        }
        const double r = exp(m[i] - m_new);
        double bsum = 0.0;
        for (size_t j = 0; j < nc; ++j) {
          const double e = exp(row[j] - m_new);
          row[j] = e;
          bsum += e;
          if (e > pamax) pamax = e;
        }
        ell[i] = r * ell[i] + bsum;
        m[i] = m_new;
        resc[i] = r;
      }
      /* P requantization (fp8_attention.cpp:127-143) */
      double sp;
      if (per_block) {
        sp = pamax == 0.0 ? 1.0 : pamax / 448.0;
        const double inv = 1.0 / sp;
        for (size_t i = 0; i < nr * nc; ++i) pc[i] = orc_round_to(s[i] * inv, ORC_E4M3, 0);
      } else {
        sp = 1.0 / 448.0;
        for (size_t i = 0; i < nr * nc; ++i) pc[i] = orc_round_to(s[i] * 448.0, ORC_E4M3, 0);
      }
      matmul_f32(pc, nr, nc, vc + c0 * d, d, 0, acc); /* fp8_attention.cpp:158-165 */
      const double gscale = sp * svv;
      for (size_t i = 0; i < nr; ++i)
        for (size_t j = 0; j < d; ++j) {
          const double gv = (double)acc[i * d + j] * (1.0 * 1.0);
          oacc[i * d + j] = to_f32(to_f32(oacc[i * d + j] * resc[i]) + to_f32(gv * gscale));
        }
    }
    for (size_t i = 0; i < nr; ++i) { /* fp8_attention.cpp:167-178 */
      if (ell[i] > 0.0) {
        const double inv = 1.0 / ell[i];
        for (size_t j = 0; j < d; ++j) o[(r0 + i) * d + j] = oacc[i * d + j] * inv;
        lse[r0 + i] = m[i] + log(ell[i]);
      } else {
        for (size_t j = 0; j < d; ++j) o[(r0 + i) * d + j] = 0.0;
        lse[r0 + i] = -INFINITY;
      }
    }
  }
  free(q), free(k), free(qc), free(kc), free(vc), free(sq), free(sk), free(sv), free(acc),
      free(s), free(pc), free(oacc), free(m), free(ell), free(resc);
  return rc;
}

/*
 * oracle.c -- plain, slow, obviously-correct CPU reference (TEST INFRASTRUCTURE).
 * See oracle.h for the contract and the paper passages each function follows.
 * Compiled with -O2 -ffp-contract=off -fno-fast-math -fopenmp (see oracle/build.py).
 * Shares no code with the CUDA path.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NT(t) ((t) > 0 ? (t) : 1)
#ifdef _OPENMP
#define OMP_THREADS(t) num_threads((t) > 0 ? (t) : omp_get_max_threads())
#else
#define OMP_THREADS(t)
#endif

/* ------------------------------------------------------------------ fp16 <-> fp64 */

double oracle_f16_to_f64(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 0x1f;
  int m = h & 0x3ff;
  double v;
  if (e == 0) {
    v = ldexp((double)m, -24); /* subnormal: m * 2^-24 */
  } else if (e == 31) {
    v = m ? NAN : INFINITY;
  } else {
    v = ldexp((double)(1024 + m), e - 25); /* (1.m) * 2^(e-15) */
  }
  return sign ? -v : v;
}

/* Round-to-nearest-even conversion fp64 -> fp16.  All scalings below are by powers
 * of two (exact); rint() rounds half to even in the default rounding mode. */
uint16_t oracle_f64_to_f16(double v) {
  uint16_t sign = signbit(v) ? 0x8000 : 0;
  double a = fabs(v);
  if (isnan(v)) return 0x7e00;
  if (a >= 65520.0) return sign | 0x7c00; /* 65520 is the tie between 65504 and 2^16 */
  if (a < ldexp(1.0, -14)) {
    double q = rint(a * 16777216.0); /* units of 2^-24; q may reach 1024 = min normal */
    return sign | (uint16_t)q;
  }
  int e;
  frexp(a, &e);        /* a = f * 2^e, f in [0.5, 1) */
  e -= 1;              /* a = g * 2^e, g in [1, 2)   */
  double m = rint(ldexp(a, 10 - e)); /* 11-bit significand in [1024, 2048] */
  if (m == 2048.0) { m = 1024.0; e += 1; }
  if (e > 15) return sign | 0x7c00;
  return sign | (uint16_t)(((e + 15) << 10) | ((int)m - 1024));
}

/* ------------------------------------------------------------------ O-1 quantize */

/* Round-half-to-even of the exact rational n/d, d > 0, n >= 0 (integers). */
static int64_t rhe_div(int64_t n, int64_t d) {
  int64_t q = n / d, r = n - q * d;
  if (2 * r > d || (2 * r == d && (q & 1))) q += 1;
  return q;
}

/* One row at b bits, qmax = 2^(b-1) - 1: x' = clip(x); a = max|x'|; q = rhe(qmax x'/a)
 * exactly; scale = fl32(a/qmax).  fp16 values are integers times 2^-24, so qmax x'/a =
 * qmax X/A with X, A integers (< 2^41; qmax X < 2^48 for b = 8). */
static void quantize_row_q(const uint16_t* x, int64_t cols, double clip, int qmax, int8_t* q, float* scale) {
  double amax = 0.0;
  for (int64_t j = 0; j < cols; ++j) {
    double v = oracle_f16_to_f64(x[j]);
    if (clip > 0.0) v = v > clip ? clip : (v < -clip ? -clip : v);
    if (fabs(v) > amax) amax = fabs(v);
  }
  if (amax == 0.0) { /* degenerate token: scale 1, all codes 0 (R5) */
    memset(q, 0, (size_t)cols);
    *scale = 1.0f;
    return;
  }
  int64_t A = (int64_t)ldexp(amax, 24);
  for (int64_t j = 0; j < cols; ++j) {
    double v = oracle_f16_to_f64(x[j]);
    if (clip > 0.0) v = v > clip ? clip : (v < -clip ? -clip : v);
    int64_t X = (int64_t)ldexp(fabs(v), 24);
    int64_t c = rhe_div((int64_t)qmax * X, A);
    if (v < 0) c = -c;
    if (c > qmax) c = qmax; /* clamp to [-2^(b-1), 2^(b-1)-1]; never binds */
    if (c < -qmax - 1) c = -qmax - 1;
    q[j] = (int8_t)c;
  }
  *scale = (float)amax / (float)qmax; /* IEEE fp32 division, correctly rounded (R6) */
}

static void quantize_row(const uint16_t* x, int64_t cols, double clip, int8_t* q, float* scale) {
  quantize_row_q(x, cols, clip, 7, q, scale);
}

static void pack_row(const int8_t* q, int64_t cols, uint8_t* out) {
  for (int64_t j = 0; j < (cols + 1) / 2; ++j) {
    uint8_t lo = (uint8_t)(q[2 * j] & 0xF);
    uint8_t hi = (2 * j + 1 < cols) ? (uint8_t)(q[2 * j + 1] & 0xF) : 0;
    out[j] = (uint8_t)(lo | (hi << 4));
  }
}

static int clip_is_f16(float clip) {
  if (clip == 0.0f) return 1;
  if (!(clip > 0.0f)) return 0;
  return oracle_f16_to_f64(oracle_f64_to_f16((double)clip)) == (double)clip;
}

int oracle_quantize_rows(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                         float clip, uint8_t* codes, float* scales, int threads) {
  if (rows < 0 || cols < 0 || ld_x < cols || !clip_is_f16(clip)) return -1;
  int64_t pb = (cols + 1) / 2;
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t r = 0; r < rows; ++r) {
    int8_t* q = (int8_t*)malloc((size_t)(cols > 0 ? cols : 1));
    quantize_row(x + r * ld_x, cols, (double)clip, q, &scales[r]);
    pack_row(q, cols, codes + r * pb);
    free(q);
  }
  return 0;
}

int oracle_quantize_rows_i8(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                            float clip, int8_t* codes, float* scales, int threads) {
  if (rows < 0 || cols < 0 || ld_x < cols || !clip_is_f16(clip)) return -1;
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t r = 0; r < rows; ++r) quantize_row_q(x + r * ld_x, cols, (double)clip, 127, codes + r * cols, &scales[r]);
  return 0;
}

/* O-15: asymmetric per-row INT4 (readings R17, R18).  x_zero = min(x'),
 * D = max(x') - min(x') (exact), q = rhe(15 (x' - x_zero) / D) exactly in [0, 15] (integers in
 * units of 2^-24: 15 (X - Z) < 2^46), scale = fl32(fl64(D) / 15) (fp64 division, then fp32);
 * constant row -> scale 1, codes 0, zero = the constant.  Codes packed as
 * unsigned nibbles, low nibble = even index. */
/* One row of O-15: codes packed two per byte (low nibble = even column), scale, zero. */
static void quantize_row_asym(const uint16_t* xr, int64_t cols, uint8_t* out, float* scale, float* zero) {
  int64_t pb = (cols + 1) / 2;
  double mn = oracle_f16_to_f64(xr[0]), mx = mn;
  for (int64_t j = 1; j < cols; ++j) {
    double v = oracle_f16_to_f64(xr[j]);
    if (v < mn) mn = v;
    if (v > mx) mx = v;
  }
  *zero = (float)mn;
  memset(out, 0, (size_t)pb);
  if (mx == mn) {
    *scale = 1.0f;
    return;
  }
  int64_t Dq = (int64_t)ldexp(mx - mn, 24);  /* exact: fp16 values are multiples of 2^-24 */
  for (int64_t j = 0; j < cols; ++j) {
    int64_t Xq = (int64_t)ldexp(oracle_f16_to_f64(xr[j]) - mn, 24);
    int64_t c = rhe_div(15 * Xq, Dq);
    if (c > 15) c = 15;  /* clamp to [0, 2^b - 1] (R17); never binds */
    out[j / 2] |= (uint8_t)((c & 0xF) << (4 * (j & 1)));
  }
  *scale = (float)((mx - mn) / 15.0);
}

int oracle_quantize_rows_asym(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                              uint8_t* codes, float* scales, float* zeros, int threads) {
  if (rows < 0 || cols <= 0 || ld_x < cols) return -1;
  int64_t pb = (cols + 1) / 2;
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t r = 0; r < rows; ++r) quantize_row_asym(x + r * ld_x, cols, codes + r * pb, &scales[r], &zeros[r]);
  return 0;
}

/* ------------------------------------------------------------------ O-2 pack */

int oracle_pack_int4(const int8_t* q, int64_t rows, int64_t cols, uint8_t* packed, int64_t* bad) {
  for (int64_t i = 0; i < rows * cols; ++i) {
    if (q[i] < -8 || q[i] > 7) {
      if (bad) *bad = i;
      return -1;
    }
  }
  for (int64_t r = 0; r < rows; ++r) pack_row(q + r * cols, cols, packed + r * ((cols + 1) / 2));
  return 0;
}

static int8_t nib(uint8_t v) { return (int8_t)((v & 0x8) ? (int)v - 16 : (int)v); }

void oracle_unpack_int4(const uint8_t* packed, int64_t rows, int64_t cols, int8_t* q) {
  int64_t pb = (cols + 1) / 2;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; ++j) {
      uint8_t b = packed[r * pb + j / 2];
      q[r * cols + j] = nib((j & 1) ? (uint8_t)(b >> 4) : (uint8_t)(b & 0xF));
    }
}

/* ------------------------------------------------------------------ O-4 GEMM */

int oracle_gemm_i32(const uint8_t* a_codes, const uint8_t* w_codes, int64_t M, int64_t N,
                    int64_t K, int32_t* acc, int threads) {
  int8_t* qa = (int8_t*)malloc((size_t)(M * K > 0 ? M * K : 1));
  int8_t* qw = (int8_t*)malloc((size_t)(N * K > 0 ? N * K : 1));
  oracle_unpack_int4(a_codes, M, K, qa);
  oracle_unpack_int4(w_codes, N, K, qw);
  int overflow = 0;
#pragma omp parallel for schedule(static) OMP_THREADS(threads) reduction(| : overflow)
  for (int64_t m = 0; m < M; ++m) {
    for (int64_t n = 0; n < N; ++n) {
      int64_t s = 0;
      for (int64_t k = 0; k < K; ++k) s += (int64_t)qa[m * K + k] * (int64_t)qw[n * K + k];
      if (s > INT32_MAX || s < INT32_MIN) overflow = 1;
      acc[m * N + n] = (int32_t)s;
    }
  }
  free(qa);
  free(qw);
  return overflow ? -1 : 0;
}

/* O-12: the same exact sum over int8 codes (no unpacking). */
static int gemm_i32_q(const int8_t* qa, const int8_t* qw, int64_t M, int64_t N, int64_t K, int32_t* acc,
                      int threads) {
  int overflow = 0;
#pragma omp parallel for schedule(static) OMP_THREADS(threads) reduction(| : overflow)
  for (int64_t m = 0; m < M; ++m) {
    for (int64_t n = 0; n < N; ++n) {
      int64_t s = 0;
      for (int64_t k = 0; k < K; ++k) s += (int64_t)qa[m * K + k] * (int64_t)qw[n * K + k];
      if (s > INT32_MAX || s < INT32_MIN) overflow = 1;
      acc[m * N + n] = (int32_t)s;
    }
  }
  return overflow ? -1 : 0;
}

int oracle_gemm_i32_i8(const int8_t* a_codes, const int8_t* w_codes, int64_t M, int64_t N, int64_t K,
                       int32_t* acc, int threads) {
  if (M < 0 || N < 0 || K < 0) return -1;
  return gemm_i32_q(a_codes, w_codes, M, N, K, acc, threads);
}

/* ------------------------------------------------------------------ O-5..O-7 */

static double gelu_erf(double t) { return 0.5 * t * (1.0 + erf(t / sqrt(2.0))); }

/* Dequant + bias + epilogue over an exact accumulator, requantizing to qmax = 7 (codes
 * packed two per byte into out_codes4) or qmax = 127 (int8 codes into out_codes8). */
static int linear_epilogue(const int32_t* acc, const double* dacc, const float* a_scales, const float* w_scales,
                           int64_t M, int64_t N, int epi_kind, const uint16_t* bias,
                           const uint16_t* residual, const uint16_t* gamma, const uint16_t* beta,
                           double ln_eps, float clip, int32_t* out_i32, uint16_t* out_f16,
                           int qmax, uint8_t* out_codes4, int8_t* out_codes8, float* out_scales,
                           float* out_zeros, int threads) {
  int64_t pb = (N + 1) / 2;
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t m = 0; m < M; ++m) {
    double* t = (double*)malloc((size_t)N * sizeof(double));
    uint16_t* y = (uint16_t*)malloc((size_t)N * sizeof(uint16_t));
    int8_t* q = (int8_t*)malloc((size_t)N);
    for (int64_t n = 0; n < N; ++n) {
      /* dequantize with the token x channel scales, add bias */
      t[n] = (dacc ? dacc[m * N + n] : (double)acc[m * N + n] * (double)a_scales[m] * (double)w_scales[n]) +
             (bias ? oracle_f16_to_f64(bias[n]) : 0.0);
    }
    switch (epi_kind) {
      case ORACLE_EPI_I32:
        memcpy(out_i32 + m * N, acc + m * N, (size_t)N * sizeof(int32_t));
        break;
      case ORACLE_EPI_F16:
        for (int64_t n = 0; n < N; ++n) out_f16[m * N + n] = oracle_f64_to_f16(t[n]);
        break;
      case ORACLE_EPI_GELU_Q4:
        for (int64_t n = 0; n < N; ++n) y[n] = oracle_f64_to_f16(gelu_erf(t[n]));
        if (out_f16) memcpy(out_f16 + m * N, y, (size_t)N * sizeof(uint16_t));
        if (out_zeros) { /* asymmetric requant (NEXT-3): O-15 on the fp16 row */
          quantize_row_asym(y, N, out_codes4 + m * pb, &out_scales[m], &out_zeros[m]);
          break;
        }
        quantize_row_q(y, N, (double)clip, qmax, q, &out_scales[m]);
        if (qmax == 7) pack_row(q, N, out_codes4 + m * pb);
        else memcpy(out_codes8 + m * N, q, (size_t)N);
        break;
      case ORACLE_EPI_RESLN_Q4: {
        double mu = 0.0, var = 0.0;
        for (int64_t n = 0; n < N; ++n) {
          t[n] += oracle_f16_to_f64(residual[m * N + n]); /* z = t + residual */
          mu += t[n];
        }
        mu /= (double)N;
        for (int64_t n = 0; n < N; ++n) var += (t[n] - mu) * (t[n] - mu);
        var /= (double)N; /* biased variance */
        double rstd = 1.0 / sqrt(var + ln_eps);
        for (int64_t n = 0; n < N; ++n)
          y[n] = oracle_f64_to_f16((t[n] - mu) * rstd * oracle_f16_to_f64(gamma[n]) +
                                   oracle_f16_to_f64(beta[n]));
        memcpy(out_f16 + m * N, y, (size_t)N * sizeof(uint16_t));
        if (out_zeros) {
          quantize_row_asym(y, N, out_codes4 + m * pb, &out_scales[m], &out_zeros[m]);
          break;
        }
        quantize_row_q(y, N, (double)clip, qmax, q, &out_scales[m]);
        if (qmax == 7) pack_row(q, N, out_codes4 + m * pb);
        else memcpy(out_codes8 + m * N, q, (size_t)N);
        break;
      }
      default:
        break;
    }
    free(t);
    free(y);
    free(q);
  }
  return (epi_kind >= ORACLE_EPI_I32 && epi_kind <= ORACLE_EPI_RESLN_Q4) ? 0 : -1;
}

static int epilogue_args_ok(int64_t M, int64_t N, int64_t K, int epi_kind, const uint16_t* residual,
                            const uint16_t* gamma, const uint16_t* beta, float clip, const int32_t* out_i32,
                            const uint16_t* out_f16, const void* out_codes, const float* out_scales) {
  if (M < 0 || N <= 0 || K <= 0 || !clip_is_f16(clip)) return 0;
  if (epi_kind == ORACLE_EPI_I32 && !out_i32) return 0;
  if (epi_kind == ORACLE_EPI_F16 && !out_f16) return 0;
  if (epi_kind == ORACLE_EPI_GELU_Q4 && (!out_codes || !out_scales)) return 0;
  if (epi_kind == ORACLE_EPI_RESLN_Q4 && (!out_codes || !out_scales || !out_f16 || !residual || !gamma || !beta))
    return 0;
  return 1;
}

int oracle_w4a4_linear(const uint8_t* a_codes, const float* a_scales,
                       const uint8_t* w_codes, const float* w_scales,
                       int64_t M, int64_t N, int64_t K, int epi_kind,
                       const uint16_t* bias, const uint16_t* residual,
                       const uint16_t* gamma, const uint16_t* beta, double ln_eps, float clip,
                       int32_t* out_i32, uint16_t* out_f16, uint8_t* out_codes, float* out_scales,
                       int threads) {
  if (!epilogue_args_ok(M, N, K, epi_kind, residual, gamma, beta, clip, out_i32, out_f16, out_codes, out_scales))
    return -1;
  int32_t* acc = (int32_t*)malloc((size_t)(M * N > 0 ? M * N : 1) * sizeof(int32_t));
  int rc = oracle_gemm_i32(a_codes, w_codes, M, N, K, acc, threads);
  if (!rc)
    rc = linear_epilogue(acc, NULL, a_scales, w_scales, M, N, epi_kind, bias, residual, gamma, beta, ln_eps, clip,
                         out_i32, out_f16, 7, out_codes, NULL, out_scales, NULL, threads);
  free(acc);
  return rc;
}

int oracle_w8a8_linear(const int8_t* a_codes, const float* a_scales, const int8_t* w_codes,
                       const float* w_scales, int64_t M, int64_t N, int64_t K, int epi_kind,
                       const uint16_t* bias, const uint16_t* residual, const uint16_t* gamma,
                       const uint16_t* beta, double ln_eps, float clip, int32_t* out_i32,
                       uint16_t* out_f16, int8_t* out_codes, float* out_scales, int threads) {
  if (!epilogue_args_ok(M, N, K, epi_kind, residual, gamma, beta, clip, out_i32, out_f16, out_codes, out_scales))
    return -1;
  int32_t* acc = (int32_t*)malloc((size_t)(M * N > 0 ? M * N : 1) * sizeof(int32_t));
  int rc = gemm_i32_q(a_codes, w_codes, M, N, K, acc, threads);
  if (!rc)
    rc = linear_epilogue(acc, NULL, a_scales, w_scales, M, N, epi_kind, bias, residual, gamma, beta, ln_eps, clip,
                         out_i32, out_f16, 127, NULL, out_codes, out_scales, NULL, threads);
  free(acc);
  return rc;
}

/* O-14: the unquantized (FP16) linear of a per-part strategy: t = sum_k a w in fp64 over the
 * fp16 operands, then the O-5..O-7 epilogues (INT4 requant for the *_Q4 kinds). */
int oracle_f16_linear(const uint16_t* a, const uint16_t* w, int64_t M, int64_t N, int64_t K, int epi_kind,
                      const uint16_t* bias, const uint16_t* residual, const uint16_t* gamma,
                      const uint16_t* beta, double ln_eps, float clip, uint16_t* out_f16,
                      uint8_t* out_codes, float* out_scales, int threads) {
  if (epi_kind == ORACLE_EPI_I32) return -1;
  if (!epilogue_args_ok(M, N, K, epi_kind, residual, gamma, beta, clip, NULL, out_f16, out_codes, out_scales))
    return -1;
  double* dacc = (double*)malloc((size_t)(M * N > 0 ? M * N : 1) * sizeof(double));
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n = 0; n < N; ++n) {
      double sacc = 0.0;
      for (int64_t k = 0; k < K; ++k) sacc += oracle_f16_to_f64(a[m * K + k]) * oracle_f16_to_f64(w[n * K + k]);
      dacc[m * N + n] = sacc;
    }
  int rc = linear_epilogue(NULL, dacc, NULL, NULL, M, N, epi_kind, bias, residual, gamma, beta, ln_eps, clip, NULL,
                           out_f16, 7, out_codes, NULL, out_scales, NULL, threads);
  free(dacc);
  return rc;
}

/* O-16: W4A4 linear with asymmetric activations: the dequantized activation is
 * scale * qa + zero, so  t = sw[n] (sa[m] sum_k qa qw + za[m] sum_k qw[n,k]) + b[n]  (fp64),
 * qa unsigned [0, 15], qw signed (symmetric per output channel).  Epilogues as O-4..O-7 (I32:
 * acc = sum qa qw); the requantizing kinds (GELU_Q4, RESLN_Q4) code their fp16 output with the
 * asymmetric quantizer O-15 (codes, scales, zeros) when out_zeros is given -- the activations
 * of an asymmetric layer (NEXT-3) -- else with the symmetric O-1. */
int oracle_w4a4_asym_linear(const uint8_t* a_codes, const float* a_scales, const float* a_zeros,
                            const uint8_t* w_codes, const float* w_scales, int64_t M, int64_t N, int64_t K,
                            int epi_kind, const uint16_t* bias, const uint16_t* residual, const uint16_t* gamma,
                            const uint16_t* beta, double ln_eps, int32_t* out_i32, uint16_t* out_f16,
                            uint8_t* out_codes, float* out_scales, float* out_zeros, int threads) {
  if (!epilogue_args_ok(M, N, K, epi_kind, residual, gamma, beta, 0.0f, out_i32, out_f16, out_codes, out_scales))
    return -1;
  int64_t pb = (K + 1) / 2;
  uint8_t* qa = (uint8_t*)malloc((size_t)(M * K > 0 ? M * K : 1));
  int8_t* qw = (int8_t*)malloc((size_t)(N * K));
  int32_t* acc = (int32_t*)malloc((size_t)(M * N > 0 ? M * N : 1) * sizeof(int32_t));
  double* dacc = (double*)malloc((size_t)(M * N > 0 ? M * N : 1) * sizeof(double));
  for (int64_t m = 0; m < M; ++m)
    for (int64_t k = 0; k < K; ++k) qa[m * K + k] = (uint8_t)((a_codes[m * pb + k / 2] >> (4 * (k & 1))) & 0xF);
  oracle_unpack_int4(w_codes, N, K, qw);
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n = 0; n < N; ++n) {
      int64_t s = 0, cs = 0;
      for (int64_t k = 0; k < K; ++k) {
        s += (int64_t)qa[m * K + k] * (int64_t)qw[n * K + k];
        cs += qw[n * K + k];
      }
      acc[m * N + n] = (int32_t)s;
      dacc[m * N + n] = (double)w_scales[n] * ((double)a_scales[m] * (double)s + (double)a_zeros[m] * (double)cs);
    }
  int rc = linear_epilogue(acc, dacc, NULL, NULL, M, N, epi_kind, bias, residual, gamma, beta, ln_eps, 0.0f, out_i32,
                           out_f16, 7, out_codes, NULL, out_scales, out_zeros, threads);
  free(qa);
  free(qw);
  free(acc);
  free(dacc);
  return rc;
}

/* O-17: l1 Pair-(2:4) pruning ("N zero-entries for every M elements",
 * 268-270: "prunes those small absolute value to be zero while keeping those large weight
 * value untouched"), applied before quantization (P => Q): in every group of
 * four consecutive elements of a row the two largest |w| are kept (ties: the lower index) and
 * the other two set to +0.  The sparse linear is then O-4/O-5 on the pruned, quantized
 * weights (zeros included) -- no new arithmetic. */
int oracle_prune_24(const uint16_t* w, int64_t N, int64_t K, uint16_t* out) {
  if (N < 0 || K <= 0 || K % 4) return -1;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t g = 0; g < K / 4; ++g) {
      const uint16_t* v = w + n * K + 4 * g;
      double a[4];
      for (int j = 0; j < 4; ++j) a[j] = fabs(oracle_f16_to_f64(v[j]));
      for (int j = 0; j < 4; ++j) {
        int beaten = 0; /* elements ranked above j: larger |w|, or equal with a lower index */
        for (int k = 0; k < 4; ++k) beaten += (a[k] > a[j]) || (a[k] == a[j] && k < j);
        out[n * K + 4 * g + j] = beaten >= 2 ? (uint16_t)0 : v[j];
      }
    }
  return 0;
}

/* ------------------------------------------------------------------ O-8 attention */

int oracle_attention(const uint16_t* qkv, int64_t B, int64_t S, int heads, int head_dim,
                     uint16_t* ctx_f16, uint8_t* ctx_codes, float* ctx_scales, int threads) {
  if (B < 0 || S <= 0 || heads <= 0 || head_dim <= 0) return -1;
  int64_t h = (int64_t)heads * head_dim, ld = 3 * h;
  int64_t T = B * S;
  uint16_t* ctx = (uint16_t*)malloc((size_t)(T * h > 0 ? T * h : 1) * sizeof(uint16_t));
  double scale = 1.0 / sqrt((double)head_dim);
#pragma omp parallel for schedule(static) OMP_THREADS(threads)
  for (int64_t bi = 0; bi < B * (int64_t)heads; ++bi) {
    int64_t b = bi / heads, j = bi % heads;
    double* p = (double*)malloc((size_t)S * sizeof(double));
    for (int64_t i = 0; i < S; ++i) {
      const uint16_t* qrow = qkv + (b * S + i) * ld + j * head_dim;
      double mx = -INFINITY;
      for (int64_t k = 0; k < S; ++k) {
        const uint16_t* krow = qkv + (b * S + k) * ld + h + j * head_dim;
        double s = 0.0;
        for (int d = 0; d < head_dim; ++d) s += oracle_f16_to_f64(qrow[d]) * oracle_f16_to_f64(krow[d]);
        p[k] = s * scale;
        if (p[k] > mx) mx = p[k];
      }
      double sum = 0.0;
      for (int64_t k = 0; k < S; ++k) { p[k] = exp(p[k] - mx); sum += p[k]; }
      for (int d = 0; d < head_dim; ++d) {
        double o = 0.0;
        for (int64_t k = 0; k < S; ++k)
          o += p[k] * oracle_f16_to_f64(qkv[(b * S + k) * ld + 2 * h + j * head_dim + d]);
        ctx[(b * S + i) * h + j * head_dim + d] = oracle_f64_to_f16(o / sum);
      }
    }
    free(p);
  }
  if (ctx_f16) memcpy(ctx_f16, ctx, (size_t)(T * h) * sizeof(uint16_t));
  int rc = oracle_quantize_rows(ctx, T, h, h, 0.0f, ctx_codes, ctx_scales, threads);
  free(ctx);
  return rc;
}

/* ------------------------------------------------------------------ O-9 layer */

int oracle_encoder_layer(const oracle_layer_cfg* cfg, const oracle_layer_weights* w,
                         int64_t B, int64_t S, const uint16_t* h_in, const uint8_t* hq_in,
                         const float* hs_in, uint16_t* h_out, uint8_t* hq_out, float* hs_out,
                         const oracle_taps* taps, int threads) {
  int64_t M = B * S, h = cfg->hidden, f = cfg->ffn;
  if ((int64_t)cfg->heads * cfg->head_dim != h) return -1;
  uint16_t* qkv = (uint16_t*)malloc((size_t)(M * 3 * h) * 2);
  uint16_t* ctx = (uint16_t*)malloc((size_t)(M * h) * 2);
  uint8_t* cq = (uint8_t*)malloc((size_t)(M * h / 2));
  float* cs = (float*)malloc((size_t)M * 4);
  uint16_t* h1 = (uint16_t*)malloc((size_t)(M * h) * 2);
  uint8_t* h1q = (uint8_t*)malloc((size_t)(M * h / 2));
  float* h1s = (float*)malloc((size_t)M * 4);
  uint16_t* ff = (uint16_t*)malloc((size_t)(M * f) * 2);
  uint8_t* fq = (uint8_t*)malloc((size_t)(M * f / 2));
  float* fs = (float*)malloc((size_t)M * 4);
  int rc = 0;
  rc |= oracle_w4a4_linear(hq_in, hs_in, w->wqkv, w->sqkv, M, 3 * h, h, ORACLE_EPI_F16, w->bqkv,
                           NULL, NULL, NULL, 0.0, 0.0f, NULL, qkv, NULL, NULL, threads);
  rc |= oracle_attention(qkv, B, S, cfg->heads, cfg->head_dim, ctx, cq, cs, threads);
  rc |= oracle_w4a4_linear(cq, cs, w->wo, w->so, M, h, h, ORACLE_EPI_RESLN_Q4, w->bo, h_in,
                           w->ln1_g, w->ln1_b, cfg->ln_eps, 0.0f, NULL, h1, h1q, h1s, threads);
  rc |= oracle_w4a4_linear(h1q, h1s, w->w1, w->s1, M, f, h, ORACLE_EPI_GELU_Q4, w->b1, NULL, NULL,
                           NULL, 0.0, 0.0f, NULL, ff, fq, fs, threads);
  rc |= oracle_w4a4_linear(fq, fs, w->w2, w->s2, M, h, f, ORACLE_EPI_RESLN_Q4, w->b2, h1,
                           w->ln2_g, w->ln2_b, cfg->ln_eps, 0.0f, NULL, h_out, hq_out, hs_out,
                           threads);
  if (taps) {
    if (taps->qkv) memcpy(taps->qkv, qkv, (size_t)(M * 3 * h) * 2);
    if (taps->ctx) memcpy(taps->ctx, ctx, (size_t)(M * h) * 2);
    if (taps->ctx_codes) memcpy(taps->ctx_codes, cq, (size_t)(M * h / 2));
    if (taps->ctx_scales) memcpy(taps->ctx_scales, cs, (size_t)M * 4);
    if (taps->h1) memcpy(taps->h1, h1, (size_t)(M * h) * 2);
    if (taps->h1_codes) memcpy(taps->h1_codes, h1q, (size_t)(M * h / 2));
    if (taps->h1_scales) memcpy(taps->h1_scales, h1s, (size_t)M * 4);
    if (taps->ffn1) memcpy(taps->ffn1, ff, (size_t)(M * f) * 2);
    if (taps->f_codes) memcpy(taps->f_codes, fq, (size_t)(M * f / 2));
    if (taps->f_scales) memcpy(taps->f_scales, fs, (size_t)M * 4);
  }
  free(qkv); free(ctx); free(cq); free(cs); free(h1); free(h1q); free(h1s);
  free(ff); free(fq); free(fs);
  return rc ? -1 : 0;
}

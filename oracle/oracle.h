/*
 * oracle.h -- plain, slow, CPU reference for the W4A4 encoder hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product
 * path (paper_2301_12017_b200/) never links, imports or executes anything here, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Every function follows a passage of the paper (PAPER.md = /root/reference/PAPER.md
 * of arXiv 2301.12017; SPEC.md is the CPU-program spec written from it).  Where the
 * paper is garbled or silent the reading adopted is the one listed in DESIGN.md
 * "Readings" (R1..R17), cited by number below.
 *
 * Conventions
 *   - fp16 values are passed as their raw IEEE-754 binary16 bit patterns (uint16_t).
 *   - Floating point inside the oracle is fp64 (double); integers are int64.  Results
 *     are rounded once, to fp16 round-to-nearest-even, where the method stores fp16.
 *   - Packed INT4: byte j of a row holds element 2j in the low nibble and 2j+1 in
 *     the high nibble, two's complement (reading R9).
 *   - All pointers are host memory owned by the caller.  `threads` <= 0 means "use
 *     the OpenMP default".
 *
 * Parity pins are in tests/test_oracle_*.py; nothing here is "parity unpinned"
 * except oracle_encoder_stack (L > 1 layers).
 */
#ifndef Q4_ORACLE_H
#define Q4_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* fp16 helpers (exposed so the tests can pin them against numpy's float16). */
double   oracle_f16_to_f64(uint16_t h);
uint16_t oracle_f64_to_f16(double v);

/* O-1  Symmetric per-row INT4 quantization.
 * PAPER.md:703-708 (App. "Quantization", symmetric equation) with S = amax/7
 * (reading R1), rounding half-to-even (R2), exact evaluation of x/S (R3),
 * per-token / per-output-channel rows (R7, R8), optional
 * activation clip (R10), all-zero row -> scale 1, codes 0 (R5).
 *   x      [rows, ld_x] fp16 bits, row-major; only the first `cols` of each row used
 *   clip   0 = no clip, else clamp x to [-clip, clip] first (clip fp16-representable)
 *   codes  [rows, ceil(cols/2)] packed nibbles (odd cols: high nibble of last byte 0)
 *   scales [rows] fp32 = fl32(amax / 7)
 * Returns 0, or -1 if clip is not fp16-representable / args invalid. */
int oracle_quantize_rows(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                         float clip, uint8_t* codes, float* scales, int threads);

/* O-2  pack / unpack.  pack returns -1 (and writes the
 * offending flat index to *bad) if a value is outside [-8, 7]. */
int  oracle_pack_int4(const int8_t* q, int64_t rows, int64_t cols, uint8_t* packed, int64_t* bad);
void oracle_unpack_int4(const uint8_t* packed, int64_t rows, int64_t cols, int8_t* q);

/* O-4  exact integer GEMM: acc[m,n] = sum_k qa[m,k] * qw[n,k]
 * a_codes [M, K/2] packed, w_codes [N, K/2] packed (nn.Linear [out,in] orientation),
 * accumulation in int64, checked to fit int32.  Returns -1 on overflow. */
int oracle_gemm_i32(const uint8_t* a_codes, const uint8_t* w_codes, int64_t M, int64_t N,
                    int64_t K, int32_t* acc, int threads);

/* Epilogue kinds (mirror of include/q4.h, restated here so the two share nothing). */
enum { ORACLE_EPI_I32 = 0, ORACLE_EPI_F16 = 1, ORACLE_EPI_GELU_Q4 = 2, ORACLE_EPI_RESLN_Q4 = 3 };

/* O-5..O-7  W4A4 linear with fused epilogue ("fuse the
 * dequantization operation with the INT4 GEMM", "fuse the quantization operation
 * ... with its previous element-bias-add, GELU, or layer normalization").
 *   t[m,n]  = acc[m,n] * a_scales[m] * w_scales[n] + bias[n]          (fp64)
 *   F16     : out_f16 = fp16(t)
 *   GELU_Q4 : y = fp16(0.5 t (1 + erf(t/sqrt2)))  (R11); out_f16 = y (optional);
 *             (out_codes, out_scales) = O-1(y) per row
 *   RESLN_Q4: z = t + residual; mu, var (biased) over the row; y = fp16((z-mu)/
 *             sqrt(var+eps) * gamma + beta)  (R12, post-LN PAPER.md:139);
 *             out_f16 = y (required); (out_codes, out_scales) = O-1(y)
 *   I32     : out_i32 = acc
 * bias may be NULL (= 0).  clip applies to the requantization (as O-1). */
int oracle_w4a4_linear(const uint8_t* a_codes, const float* a_scales,
                       const uint8_t* w_codes, const float* w_scales,
                       int64_t M, int64_t N, int64_t K, int epi_kind,
                       const uint16_t* bias, const uint16_t* residual,
                       const uint16_t* gamma, const uint16_t* beta, double ln_eps, float clip,
                       int32_t* out_i32, uint16_t* out_f16, uint8_t* out_codes, float* out_scales,
                       int threads);

/* O-8  FP16 attention glue + per-token requant.
 * qkv [B*S, 3*heads*head_dim] fp16: Q = cols [0,h), K = [h,2h), V = [2h,3h);
 * head j = cols [j*d, (j+1)*d) of each.  Scores scaled by 1/sqrt(d), softmax over all
 * S keys (no mask, R14), ctx = P V rounded to fp16, then O-1 per token over all h.
 * ctx_f16 may be NULL. */
int oracle_attention(const uint16_t* qkv, int64_t B, int64_t S, int heads, int head_dim,
                     uint16_t* ctx_f16, uint8_t* ctx_codes, float* ctx_scales, int threads);

/* O-9  One post-LN BERT encoder layer, all four linears W4A4 ("qall", PAPER.md:
 * 429-431, 467-476, R15).  Weights are given already quantized (O-3 = O-1 on W rows).
 * Every intermediate may be captured through the optional tap pointers (NULL = skip).
 *   qkv  = F16(QKV)          ctx = O-8(qkv)
 *   h1   = RESLN_Q4(O, residual h_in, ln1)
 *   f    = GELU_Q4(FFN1)
 *   h_out= RESLN_Q4(FFN2, residual h1, ln2)  */
typedef struct {
  int hidden, heads, head_dim, ffn;
  double ln_eps;
} oracle_layer_cfg;
typedef struct {
  const uint8_t *wqkv, *wo, *w1, *w2;
  const float *sqkv, *so, *s1, *s2;
  const uint16_t *bqkv, *bo, *b1, *b2, *ln1_g, *ln1_b, *ln2_g, *ln2_b;
} oracle_layer_weights;
typedef struct {
  uint16_t *qkv, *ctx, *h1, *ffn1;
  uint8_t *ctx_codes, *h1_codes, *f_codes;
  float *ctx_scales, *h1_scales, *f_scales;
} oracle_taps;
int oracle_encoder_layer(const oracle_layer_cfg* cfg, const oracle_layer_weights* w,
                         int64_t B, int64_t S, const uint16_t* h_in, const uint8_t* hq_in,
                         const float* hs_in, uint16_t* h_out, uint8_t* hq_out, float* hs_out,
                         const oracle_taps* taps, int threads);

/* O-11..O-13  W8A8 variant of the same linear ("i8-qall": the
 * paper's INT8 baseline that INT4 is measured against).  Identical definitions at
 * b = 8 bits, qmax = 2^(b-1) - 1 = 127 (PAPER.md:703-708 with reading R1 at b = 8):
 *   O-11 quantize_rows_i8: q = rhe(127 x'/a) exactly, scale = fl32(a/127); codes int8
 *        [rows, cols], one per byte (no packing)
 *   O-12 gemm_i32_i8: acc = sum_k qa qw over int8 codes, int64, checked to fit int32
 *   O-13 w8a8_linear: O-5..O-7 on that accumulator; GELU_Q4 / RESLN_Q4 kinds requantize
 *        with O-11 (int8 codes) instead of O-1 */
int oracle_quantize_rows_i8(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                            float clip, int8_t* codes, float* scales, int threads);
int oracle_gemm_i32_i8(const int8_t* a_codes, const int8_t* w_codes, int64_t M, int64_t N, int64_t K,
                       int32_t* acc, int threads);
int oracle_w8a8_linear(const int8_t* a_codes, const float* a_scales, const int8_t* w_codes,
                       const float* w_scales, int64_t M, int64_t N, int64_t K, int epi_kind,
                       const uint16_t* bias, const uint16_t* residual, const uint16_t* gamma,
                       const uint16_t* beta, double ln_eps, float clip, int32_t* out_i32,
                       uint16_t* out_f16, int8_t* out_codes, float* out_scales, int threads);

/* O-14  FP16 linear of the unquantized parts of a per-part quantization strategy
 * (SURVEY 8(f) NEXT-1): t = sum_k a[m,k] w[n,k] over fp16 operands in
 * fp64 (+ bias), then the O-5..O-7 epilogues F16 / GELU_Q4 / RESLN_Q4 (INT4 requant by O-1).
 * I32 is not defined here (-1). */
int oracle_f16_linear(const uint16_t* a, const uint16_t* w, int64_t M, int64_t N, int64_t K, int epi_kind,
                      const uint16_t* bias, const uint16_t* residual, const uint16_t* gamma,
                      const uint16_t* beta, double ln_eps, float clip, uint16_t* out_f16,
                      uint8_t* out_codes, float* out_scales, int threads);

/* O-15 / O-16  Asymmetric activation quantization (the
 * paper's "asym" rows, "slower because of the bias term" PAPER.md:499).  O-15: per row
 * x_zero = min, q = rhe(15 (x - min) / (max - min)) in [0, 15] (unsigned nibbles), scale =
 * fl32(fl64(max - min) / 15), constant row -> scale 1, codes 0 (reading R18).  O-16: the
 * linear on those codes x symmetric INT4 weights, F16 / I32 epilogues:
 * t = sw (sa acc + za colsum(qw)) + b. */
int oracle_quantize_rows_asym(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                              uint8_t* codes, float* scales, float* zeros, int threads);
int oracle_w4a4_asym_linear(const uint8_t* a_codes, const float* a_scales, const float* a_zeros,
                            const uint8_t* w_codes, const float* w_scales, int64_t M, int64_t N, int64_t K,
                            int epi_kind, const uint16_t* bias, const uint16_t* residual, const uint16_t* gamma,
                            const uint16_t* beta, double ln_eps, int32_t* out_i32, uint16_t* out_f16,
                            uint8_t* out_codes, float* out_scales, float* out_zeros, int threads);
/* O-17: l1 Pair-(2:4) pruning of fp16 rows along K (two largest |w| of every four kept). */
int oracle_prune_24(const uint16_t* w, int64_t N, int64_t K, uint16_t* out);

#ifdef __cplusplus
}
#endif
#endif

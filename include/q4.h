/*
 * q4.h -- C ABI of the B200 (sm_100a) W4A4 encoder hot path.
 *
 * Paper: arXiv 2301.12017, "Highly Optimized INT4 Encoder Inference",
 * PAPER.md:402-511, and App. A "Quantization Algorithms".
 * Readings of garbled / silent passages are numbered R1..R17 in DESIGN.md.
 *
 * Conventions (all entry points)
 *   - fp16 tensors are IEEE binary16, passed as `uint16_t*`; fp32 as `float*`.
 *   - Packed INT4 ("we pack INT4 data into INT8 tensors"): byte j of a
 *     row holds element 2j in the low nibble and 2j+1 in the high nibble, two's
 *     complement (R9).  A row of `cols` INT4 values occupies cols/2 bytes.
 *   - All matrices are row-major and contiguous unless an ld_* argument is given.
 *     Weights use the nn.Linear [out, in] orientation, i.e. [N, K]: both GEMM
 *     operands are K-major and nibble-packed along K.
 *   - Pointers are caller-owned DEVICE memory unless stated (q4_encoder_stack also
 *     accepts host memory for its input/output).  The library never allocates in
 *     these calls; scratch comes in through `workspace`, sized by *_workspace().
 *     A workspace must be ZERO-FILLED before its first use (cudaMemset): the row
 *     epilogues keep self-resetting cross-CTA rendezvous counters in it, and every
 *     completed call leaves them zero again, so no per-call reset (and no memset node
 *     in a captured graph) is needed.  The counters sit at the start of the workspace at
 *     an offset that depends on M only, so one linear workspace serves row-epilogue calls
 *     of the same M and any N / K (an encoder layer's N = hidden and N = ffn launches);
 *     a call with a different M needs its own zero-filled workspace.  A counter left
 *     non-zero (e.g. by a kernel fault) makes the next row-epilogue call trap with
 *     Q4_ECUDA instead of hanging.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are stream-ordered and asynchronous: no host synchronisation, no
 *     allocation, no host-side state change, so they can be captured in CUDA graphs
 *     (except q4_encoder_stack with host buffers, which enqueues copies).
 *   - Errors: argument validation is synchronous and returns Q4_E*; the text naming
 *     the argument, shape or coordinate is in q4_last_error() (thread-local).  A
 *     launch failure returns Q4_ECUDA; asynchronous kernel faults surface at the
 *     caller's next synchronisation.  The library never aborts the process.
 */
#ifndef Q4_H
#define Q4_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define Q4_API __attribute__((visibility("default")))
#else
#define Q4_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  Q4_OK = 0,
  Q4_EINVAL = 1,       /* bad argument value (NULL where required, bad clip, bad kind) */
  Q4_ESHAPE = 2,       /* inconsistent or unsupported dimensions                       */
  Q4_EALIGN = 3,       /* pointer / leading-dimension alignment (TMA needs 16 B)       */
  Q4_EUNSUPPORTED = 4, /* valid request this build does not implement                 */
  Q4_ECUDA = 5         /* CUDA runtime / driver error (text has cudaGetErrorString)    */
} q4_status;

/* Thread-local description of the last error of this thread ("" if none). */
Q4_API const char* q4_last_error(void);
/* Library version / build string (architecture it was compiled for). */
Q4_API const char* q4_version(void);
/* Number of kernels this process launched through the library (all threads). */
Q4_API uint64_t q4_launch_count(void);
/* Measurement only (the latency roofline of BASELINE configs[2]: "launch
 * overhead non-negligible"): launch `n` empty kernels of `ctas` CTAs x 128 threads on `stream`
 * with the same programmatic-dependent-launch attribute the encoder uses for small problems,
 * so a CUDA graph of them gives the empty-graph floor for the encoder's kernel count.
 * n in [0, 4096], ctas in [1, 1024]; Q4_EINVAL otherwise.  No memory is touched. */
Q4_API q4_status q4_launch_floor(int32_t n, int32_t ctas, void* stream);

/* ---------------------------------------------------------------------------------
 * a1/a2  Symmetric per-row INT4 quantization + packing.
 * PAPER.md:703-708 (sym. equation) with S = amax / (2^(b-1) - 1) = amax/7 (R1),
 * round half to even (R2), x/S evaluated exactly (R3): q = rint(div.rn(7x, amax)),
 * which equals the exact rational rounding for every fp16 pair (tests pin this).
 * Rows are tokens for activations ("token-wise dynamic quantization",
 * PAPER.md:520-522) or output channels for weights ("row-wise", R7).
 *   x       [rows, ld_x] fp16; the first `cols` of each row are quantized
 *   clip    0 = none; else an fp16-representable value > 0, x clamped to
 *           [-clip, clip] before the scale is taken ("Clip Values", R10)
 *   codes   [rows, cols/2] packed INT4 (output)
 *   scales  [rows] fp32 = fl32(amax/7); an all-zero row gets scale 1, codes 0 (R5)
 * Requirements: cols % 8 == 0, ld_x % 8 == 0, x 16-byte aligned, codes 4-byte aligned.
 * rows == 0 is a no-op. */
Q4_API q4_status q4_quantize_rows(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                           float clip, uint8_t* codes, float* scales, void* stream);

/* ---------------------------------------------------------------------------------
 * a3-a6  W4A4 linear: exact INT32 GEMM + fused epilogue.
 *   acc[m,n] = sum_k qa[m,k] * qw[n,k]                  (exact)
 *   t[m,n]   = acc * a_scales[m] * w_scales[n] + bias[n]   (fp32; "fuse the
 *              dequantization operation with the INT4 GEMM kernel")
 * Epilogues ("fuse the quantization operation for activation with its previous
 * element-bias-add, GELU, or layer normalization operation"):
 *   Q4_EPI_I32      out_i32 = acc                              (debug / parity tap)
 *   Q4_EPI_F16      out_f16 = fp16(t)                          (QKV projection)
 *   Q4_EPI_GELU_Q4  y = fp16(gelu_erf(t)) (R11); (out_codes, out_scales) = a1(y)
 *                   per row; out_f16 = y if non-NULL (tap)     (MLP intermediate)
 *   Q4_EPI_RESLN_Q4 z = t + residual; y = fp16(LayerNorm(z) * gamma + beta), biased
 *                   variance, eps = ln_eps (R12), post-LN;
 *                   out_f16 = y (required: next residual); (out_codes, out_scales)
 *                   = a1(y)                                    (attn-out, MLP-out)
 * The *_Q4 epilogues reduce over a whole output row; they need N <= 4096.
 */
typedef enum { Q4_EPI_I32 = 0, Q4_EPI_F16 = 1, Q4_EPI_GELU_Q4 = 2, Q4_EPI_RESLN_Q4 = 3 } q4_epi_kind;

/* GEMM mainloop variant (benchmark knob; results are identical by construction).
 *   AUTO        choose by shape (currently TCGEN05)
 *   TCGEN05     TMA -> smem nibble->int8 unpack -> tcgen05.mma kind::i8 -> TMEM
 *   MMA_SYNC_S8 legacy: cp.async -> ldmatrix -> register unpack -> mma.sync s8
 *   MMA_SYNC_S4 legacy: cp.async -> ldmatrix -> mma.sync m16n8k64 .s4 (emulated on sm_100a)
 *   TCGEN05_W8  as TCGEN05, but the weights come prepacked (epi->w_i8, q4_prepack_weights):
 *               TMA'd straight into the swizzled operand stage; only A is unpacked on chip
 *   TCGEN05_W8_1CTA  as TCGEN05_W8, never the CTA-pair (cta_group::2) mainloop that
 *               TCGEN05_W8 / AUTO pick for F16 / I32 at M % 256 == 0, M >= 8192 (the row
 *               epilogues always run 1-CTA; this reproduces their accumulators in an I32 tap)
 * AUTO uses TCGEN05_W8 when epi->w_i8 is given (faster at every measured M, 128..32768:
 * profiles/r1_gemm_sweep.jsonl), else TCGEN05.
 * The legacy variants implement Q4_EPI_I32 and Q4_EPI_F16 only. */
typedef enum { Q4_MAINLOOP_AUTO = 0, Q4_MAINLOOP_TCGEN05 = 1, Q4_MAINLOOP_MMA_SYNC_S8 = 2,
               Q4_MAINLOOP_MMA_SYNC_S4 = 3, Q4_MAINLOOP_TCGEN05_W8 = 4,
               Q4_MAINLOOP_TCGEN05_W8_1CTA = 5 } q4_mainloop;

typedef struct {
  int32_t kind;              /* q4_epi_kind                                              */
  int32_t mainloop;          /* q4_mainloop (0 = auto)                                   */
  const uint16_t* bias;      /* [N] fp16; NULL = 0                                       */
  const uint16_t* residual;  /* [M, N] fp16; RESLN only                                  */
  const uint16_t* gamma;     /* [N] fp16; RESLN only                                     */
  const uint16_t* beta;      /* [N] fp16; RESLN only                                     */
  float ln_eps;              /* RESLN; BERT uses 1e-12                                   */
  float requant_clip;        /* *_Q4: as q4_quantize_rows' clip; 0 = none                */
  int32_t* out_i32;          /* [M, N]   I32                                             */
  uint16_t* out_f16;         /* [M, N]   F16, RESLN (required); GELU_Q4 optional tap      */
  uint8_t* out_codes;        /* [M, N/2] *_Q4                                            */
  float* out_scales;         /* [M]      *_Q4                                            */
  const int8_t* w_i8;        /* optional [N, K] prepacked weights (q4_prepack_weights) of the
                                same codes as w_codes; NULL = unpack w_codes on chip       */
  float* out_zeros;          /* [M] GELU_Q4 / RESLN_Q4: non-NULL = ASYMMETRIC requant of the
                                fp16 output (NEXT-3, q4_quantize_rows_asym's
                                definition: unsigned codes, scales = (max-min)/15, zeros = min);
                                requant_clip must be 0; NULL = symmetric (a1)               */
} q4_epilogue;

/* Requirements: M >= 0; N % 32 == 0 (row epilogues N % 64 == 0); K % 32 == 0; K <= 8192
 * (the INT32 accumulator bound |acc| <= 64 K); N / tile_n <= #SMs (every CTA owns one n-block,
 * tile_n = 256 for M > 512, 64 below: N <= 37,888 resp. 9,472 on B200; larger N returns
 * Q4_EUNSUPPORTED); all pointers 16-byte aligned.  Workspace: q4_w4a4_linear_workspace bytes
 * (row epilogues: the cross-CTA exchange slots and self-resetting counters; M <= 256, every
 * kind: the split-K region -- tile counters and INT32 partial sums that several CTAs add into
 * with integer reductions, exact in any order, DESIGN.md 4.3 -- which the last CTA of each
 * tile zeroes again; zero-filled once before first use, left zeroed by every launch).  I32 /
 * F16 at M > 256 need none; a NULL / short workspace there just disables split-K. */
Q4_API size_t q4_w4a4_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t kind);
Q4_API q4_status q4_w4a4_linear(const uint8_t* a_codes, const float* a_scales, /* [M,K/2], [M] */
                         const uint8_t* w_codes, const float* w_scales, /* [N,K/2], [N] */
                         int64_t M, int64_t N, int64_t K, const q4_epilogue* epi,
                         void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * W8A8 baseline: the same linear with 8-bit codes -- the paper's
 * INT8 comparison point ("i8-qall"; INT4 vs INT8 GEMM, Fig.
 * gemm_perf).  Definitions are those above at b = 8 bits (oracle O-11..O-13):
 *
 * q4_quantize_rows_i8: PAPER.md:703-708 with S = amax/127 (R1 at b = 8), round half to
 *   even (R2), exact evaluation (R3).  codes [rows, cols] int8 (one per byte, in
 *   [-127, 127]); scales [rows] fp32 = fl32(amax/127); all-zero row -> scale 1, codes 0.
 *   Requirements as q4_quantize_rows, codes 8-byte aligned.
 *
 * q4_w8a8_linear: acc = sum_k qa[m,k] qw[n,k] exact in INT32 over int8 codes
 *   a_codes [M, K] and w_codes [N, K] (nn.Linear [out, in] orientation, K-major, no
 *   packing), then the Q4_EPI_* epilogues of q4_w4a4_linear with the requantizing kinds
 *   (GELU_Q4 / RESLN_Q4) writing int8 codes out_codes [M, N] (q4_quantize_rows_i8 of the
 *   fp16 y) and scales amax/127.  Both operands are TMA'd straight into the MMA stage
 *   (no unpack).  epi->mainloop must be AUTO or TCGEN05; epi->w_i8 is ignored.
 *   Requirements: N % 32 == 0 (row epilogues: N % 64 == 0),
 *   K % 128 == 0, K <= 131072 (|acc| <= 128^2 K < 2^31), pointers 16-byte aligned;
 *   workspace: q4_w8a8_linear_workspace (row epilogues).  Errors as q4_w4a4_linear. */
Q4_API q4_status q4_quantize_rows_i8(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                                     float clip, int8_t* codes, float* scales, void* stream);
Q4_API size_t q4_w8a8_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t kind);
Q4_API q4_status q4_w8a8_linear(const int8_t* a_codes, const float* a_scales, /* [M,K], [M] */
                                const int8_t* w_codes, const float* w_scales, /* [N,K], [N] */
                                int64_t M, int64_t N, int64_t K, const q4_epilogue* epi,
                                void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * FP16 linear for the unquantized parts of a per-part quantization strategy (SURVEY 8(f)
 * NEXT-1; "the four model parts as modular components where quantization
 * can be enabled or disabled separately").  a [M, K] and w [N, K] fp16 (nn.Linear
 * orientation), t = sum_k a w in fp32 on the tensor cores (tcgen05.mma kind::f16) + bias;
 * epilogues Q4_EPI_F16, Q4_EPI_GELU_Q4 and Q4_EPI_RESLN_Q4 exactly as q4_w4a4_linear
 * (the *_Q4 kinds still emit INT4 codes for a quantized successor, plus the fp16 output).
 * Requirements: N % 32 == 0 (row epilogues N % 64 == 0), K % 64 == 0, pointers 16-byte
 * aligned; workspace q4_f16_linear_workspace for the row epilogues. */
Q4_API size_t q4_f16_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t kind);
Q4_API q4_status q4_f16_linear(const uint16_t* a, const uint16_t* w, int64_t M, int64_t N, int64_t K,
                               const q4_epilogue* epi, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Asymmetric activation quantization (the paper's
 * "asym" rows -- "slower ... because of less required computation for bias term" for sym,
 * PAPER.md:499).  Oracle O-15 / O-16, readings R17 / R18.
 * q4_quantize_rows_asym: per row zero = min(x), q = rhe(15 (x - min) / (max - min)) in
 *   [0, 15] (exact rational; unsigned nibbles, low = even index), scale = fl32(fl64(max -
 *   min) / 15); constant row -> scale 1, codes 0, zero = the constant.  cols % 8 == 0,
 *   cols <= 4096.
 * q4_weight_code_sums: sums[n] = sum_k qw[n, k] of packed INT4 weights (offline, as float).
 * q4_w4a4_asym_linear: unsigned activation codes x signed weight codes on tcgen05 (u8 x s8),
 *   t = w_scales[n] (a_scales[m] acc + a_zeros[m] w_sums[n]) + bias[n]; all four epilogues
 *   (I32: acc = sum qa qw; F16; GELU_Q4 and RESLN_Q4 as in q4_w4a4_linear, their codes
 *   asymmetric when epi->out_zeros is set -- the asymmetric encoder layer -- else symmetric);
 *   epi->w_i8 (prepacked weights) honoured; requant_clip must be 0.  The row epilogues take
 *   a q4_w4a4_linear_workspace(M, N, K, kind) workspace (same contract); I32 / F16 none.
 * q4_attention_f16_q4_asym: q4_attention_f16_q4 with the per-token ctx codes of
 *   q4_quantize_rows_asym (codes, scales, zeros [B*S] fp32, 4-byte aligned). */
Q4_API q4_status q4_quantize_rows_asym(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x,
                                       uint8_t* codes, float* scales, float* zeros, void* stream);
Q4_API q4_status q4_weight_code_sums(const uint8_t* w_codes, int64_t N, int64_t K, float* sums,
                                     void* stream);
Q4_API q4_status q4_w4a4_asym_linear(const uint8_t* a_codes, const float* a_scales,
                                     const float* a_zeros, const uint8_t* w_codes,
                                     const float* w_scales, const float* w_sums, int64_t M, int64_t N,
                                     int64_t K, const q4_epilogue* epi, void* workspace, size_t ws_bytes,
                                     void* stream);
Q4_API q4_status q4_attention_f16_q4_asym(const uint16_t* qkv, int64_t B, int64_t S, int32_t heads,
                                          int32_t head_dim, uint16_t* ctx_f16, uint8_t* ctx_codes,
                                          float* ctx_scales, float* ctx_zeros, void* stream);

/* ---------------------------------------------------------------------------------
 * NEXT-4: W4A4 with 2:4-sparse weights -- the paper's "Pair-(2:4)" (50%)
 * semi-structured sparsity composed with INT4, pruning before quantization (P => Q) with the
 * l1 criterion.  Offline: q4_prune_24 -> q4_quantize_rows (a2) ->
 * q4_sparse24_compress; forward: q4_w4a4_sparse24_linear on the sparse tensor cores
 * (tcgen05.mma.sp kind::i8, half the weight MMA operand bytes).
 * q4_prune_24: w [N, K] fp16 rows; in every group of four consecutive k the two largest |w|
 *   are kept (ties: the lower index) and the other two set to +0.  K % 4 == 0, 8-byte aligned.
 * q4_sparse24_compress: packed INT4 codes [N, K/2] with at most two nonzero codes per group of
 *   four -> w_vals [N, K/2] int8 (16*q of the two kept codes per group, in k order; a group
 *   with fewer nonzeros keeps zero codes at its lowest free positions) + w_meta [N, K/32]
 *   uint32 (per group the nibble i0 | i1 << 2 of the kept positions, i0 < i1, eight groups per
 *   word in k order -- the tcgen05.mma.sp metadata layout).  `violations` (nullable, device
 *   int, accumulated) counts groups with more than two nonzero codes: their extra codes are
 *   dropped.  K % 256 == 0, pointers 16-byte aligned.
 * q4_w4a4_sparse24_linear: as q4_w4a4_linear (a3/a4: exact INT32 sum, then
 *   t = acc * a_scales[m] * w_scales[n] + bias[n]) with the compressed weights; epilogues F16 and
 *   I32 only.  N % 128 == 0, K % 256 == 0, K <= 8192, N / 128 <= #SMs; no workspace. */
Q4_API q4_status q4_prune_24(const uint16_t* w, int64_t N, int64_t K, uint16_t* out, void* stream);
Q4_API q4_status q4_sparse24_compress(const uint8_t* w_codes, int64_t N, int64_t K, int8_t* w_vals,
                                      uint32_t* w_meta, int32_t* violations, void* stream);
Q4_API q4_status q4_w4a4_sparse24_linear(const uint8_t* a_codes, const float* a_scales,
                                         const int8_t* w_vals, const uint32_t* w_meta,
                                         const float* w_scales, int64_t M, int64_t N, int64_t K,
                                         const q4_epilogue* epi, void* stream);

/* ---------------------------------------------------------------------------------
 * a2' Offline weight prepack (once per weight, not on the forward path): packed INT4 codes
 * w_codes [N, K/2] -> w_i8 [N, K] int8 holding 16*q in the K order of the on-chip
 * activation unpack (per 32-element group: the 16 even-k values, then the 16 odd-k).
 * The weights stay INT4-valued; only their on-device layout is
 * MMA-ready, trading 2x weight bytes for 3x less on-chip unpack work.
 * Requirements: K % 32 == 0, pointers 16-byte aligned. */
Q4_API q4_status q4_prepack_weights(const uint8_t* w_codes, int64_t N, int64_t K, int8_t* w_i8,
                                    void* stream);

/* ---------------------------------------------------------------------------------
 * a7  FP16 attention between the quantized GEMMs (the
 * pipeline keeps attention in FP16 -- "we use FP16 FlashAttention") with the
 * per-token quantize of the context fused into the same kernel.
 *   qkv        [B*S, 3*heads*head_dim] fp16 (Q | K | V column blocks, head j at
 *              columns [j*head_dim, (j+1)*head_dim) of each block)
 *   ctx        = softmax(Q K^T / sqrt(head_dim)) V, no mask (R14), rounded to fp16
 *   ctx_f16    [B*S, heads*head_dim] fp16 output (required: the kernel streams the
 *              context through it and re-reads it from L2 for the quantize)
 *   ctx_codes  [B*S, heads*head_dim/2], ctx_scales [B*S]: a1 applied per token over
 *              all heads of the fp16 ctx
 * Requirements: head_dim == 64, 1 <= S <= 128, heads*64 <= 1024. */
Q4_API q4_status q4_attention_f16_q4(const uint16_t* qkv, int64_t B, int64_t S, int32_t heads,
                              int32_t head_dim, uint16_t* ctx_f16, uint8_t* ctx_codes,
                              float* ctx_scales, void* stream);

/* ---------------------------------------------------------------------------------
 * a8  One post-LN BERT encoder layer, all four linears W4A4 ("qall",
 * PAPER.md:429-431, 483-493, R15):
 *   qkv   = linear(hq_in;  Wqkv, F16)                 [M, 3h]
 *   ctx   = attention(qkv) -> codes                   [M, h]
 *   h1    = linear(ctx;    Wo,  RESLN_Q4, res=h_in, ln1)
 *   f     = linear(h1;     W1,  GELU_Q4)              [M, ffn]
 *   h_out = linear(f;      W2,  RESLN_Q4, res=h1,   ln2)  (+ hq_out, hs_out)
 * (hq_in, hs_in) must be a1(h_in): the previous layer's RESLN_Q4 output, or
 * q4_quantize_rows for layer 0.  M = B*S.  Taps (each nullable) receive copies of the
 * intermediates for teacher-forced parity; acc_* taps cost one extra I32 GEMM each. */
typedef struct {
  int32_t hidden, heads, head_dim, ffn;
  float ln_eps;
  /* Per-part quantization strategy: bit 0 QKV
   * projection, bit 1 attention output, bit 2 MLP intermediate, bit 3 MLP output run in
   * FP16 (q4_f16_linear on the fp16 weights of the f* fields and the fp16 activations the
   * previous step already produces); 0 = all four parts quantized ("qall").  The paper's
   * best small-batch strategy "q3" (only the MLP intermediate quantized) is 0xB.  W4A4
   * entry points only (the *_w8a8 ones require 0). */
  int32_t fp16_parts;
  /* Asymmetric activations: 1 = every activation
   * quantize of the layer is q4_quantize_rows_asym's (unsigned codes, scales, zeros) -- the
   * layer-0 input, the attention ctx codes and the three requantizing epilogues -- and the four
   * linears run q4_w4a4_asym_linear with the weight code sums (cqkv/co/c1/c2).  Requires
   * fp16_parts == 0; the single-layer entry is q4_encoder_layer_asym; q4_encoder_stack(_w4a4)
   * and q4_encoder_pipeline honour it; the *_w8a8 entry points require 0. */
  int32_t asym_acts;
} q4_layer_cfg;
typedef struct {
  const uint8_t *wqkv, *wo, *w1, *w2;   /* packed [3h,h/2], [h,h/2], [ffn,h/2], [h,ffn/2] */
  const int8_t *wqkv8, *wo8, *w18, *w28; /* optional prepacked copies (q4_prepack_weights)  */
  const float *sqkv, *so, *s1, *s2;     /* per-output-channel scales                       */
  const uint16_t *bqkv, *bo, *b1, *b2;  /* fp16 biases                                      */
  const uint16_t *ln1_g, *ln1_b, *ln2_g, *ln2_b;
  const uint16_t *fqkv, *fo, *f1, *f2;  /* fp16 [N, K] weights of the FP16 parts (cfg->fp16_parts);
                                           NULL when the part is quantized               */
  const float *cqkv, *co, *c1, *c2;     /* cfg->asym_acts: per-output-channel weight code sums
                                           (q4_weight_code_sums), 16-byte aligned; else NULL  */
} q4_layer_weights;
typedef struct {
  uint16_t *qkv, *ctx, *h1, *ffn1;
  int32_t *acc_qkv, *acc_o, *acc_1, *acc_2;
  uint8_t *ctx_codes, *h1_codes, *f_codes;
  float *ctx_scales, *h1_scales, *f_scales;
  float *ctx_zeros, *h1_zeros, *f_zeros;  /* asymmetric layer: zero points of the codes above */
} q4_taps;
Q4_API size_t q4_encoder_layer_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S);
/* The asymmetric layer (cfg->asym_acts = 1): (hq_in, hs_in, hz_in) = q4_quantize_rows_asym(h_in)
 * or the previous asymmetric layer's output; writes (hq_out, hs_out, hz_out) likewise. */
Q4_API q4_status q4_encoder_layer_asym(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B,
                                       int64_t S, const uint16_t* h_in, const uint8_t* hq_in,
                                       const float* hs_in, const float* hz_in, uint16_t* h_out,
                                       uint8_t* hq_out, float* hs_out, float* hz_out, void* workspace,
                                       size_t ws_bytes, const q4_taps* taps, void* stream);
Q4_API q4_status q4_encoder_layer(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B,
                           int64_t S, const uint16_t* h_in, const uint8_t* hq_in,
                           const float* hs_in, uint16_t* h_out, uint8_t* hq_out, float* hs_out,
                           void* workspace, size_t ws_bytes, const q4_taps* taps, void* stream);

/* ---------------------------------------------------------------------------------
 * a8  L-layer encoder forward (the paper's E2E pipeline):
 * a1(h_in) once, then L x q4_encoder_layer, ping-ponging hidden states in the
 * workspace.  h_in / h_out may be HOST (pinned or pageable) or DEVICE pointers; host
 * buffers are copied with cudaMemcpyAsync on `stream` inside the call (this is the
 * end-to-end entry point).  `layers` is a host array of L weight structs (device
 * pointers inside).  All-device calls are CUDA-graph capturable. */
Q4_API size_t q4_encoder_stack_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S);
Q4_API q4_status q4_encoder_stack(const q4_layer_cfg* cfg, const q4_layer_weights* layers, int32_t L,
                           int64_t B, int64_t S, const uint16_t* h_in, uint16_t* h_out,
                           void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Pipelined serving over host buffers (the end-to-end path): nbatch batches, each B x S
 * tokens, h_in[i] / h_out[i] host pointers (pinned for overlap) of [B*S, hidden] fp16.
 * Batch i's upload (copy-in stream), forward (the caller's stream, = q4_encoder_stack) and
 * download (copy-out stream) overlap the neighbouring batches through two device input and
 * two device output buffers inside `workspace` (q4_encoder_pipeline_workspace).  The
 * caller's stream completes after the last download.  The two copy streams and their events
 * are created per call and released when the enqueued work completes, so concurrent calls
 * (distinct workspaces) are independent; not CUDA-graph capturable. */
Q4_API size_t q4_encoder_pipeline_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S);
Q4_API q4_status q4_encoder_pipeline(const q4_layer_cfg* cfg, const q4_layer_weights* layers, int32_t L,
                                     int64_t B, int64_t S, const uint16_t* const* h_in,
                                     uint16_t* const* h_out, int32_t nbatch, void* workspace,
                                     size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * W8A8 baseline of a7 / a8 (the paper's end-to-end INT8 comparison,
 * "i8-qall", Fig. e2e_i4_i8): the same layer and stack with 8-bit
 * codes throughout -- q4_quantize_rows_i8 for the layer-0 input, q4_w8a8_linear for the
 * four linears, and q4_attention_f16_q8 (as q4_attention_f16_q4, but ctx_codes [B*S, h]
 * int8 with ctx_scales = amax/127, codes 8-byte aligned).  In q4_layer_weights the
 * wqkv / wo / w1 / w2 fields then hold int8 codes [N, K] (q4_quantize_rows_i8 of the fp16
 * weights) and the *8 prepack fields are ignored; hq_in / hq_out and the code taps are
 * int8 [M, hidden] / [M, ffn].  Requirements and errors as the W4A4 entry points. */
Q4_API q4_status q4_attention_f16_q8(const uint16_t* qkv, int64_t B, int64_t S, int32_t heads,
                                     int32_t head_dim, uint16_t* ctx_f16, int8_t* ctx_codes,
                                     float* ctx_scales, void* stream);
Q4_API size_t q4_encoder_layer_w8a8_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S);
Q4_API q4_status q4_encoder_layer_w8a8(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B,
                                       int64_t S, const uint16_t* h_in, const int8_t* hq_in,
                                       const float* hs_in, uint16_t* h_out, int8_t* hq_out,
                                       float* hs_out, void* workspace, size_t ws_bytes,
                                       const q4_taps* taps, void* stream);
Q4_API size_t q4_encoder_stack_w8a8_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S);
Q4_API q4_status q4_encoder_stack_w8a8(const q4_layer_cfg* cfg, const q4_layer_weights* layers,
                                       int32_t L, int64_t B, int64_t S, const uint16_t* h_in,
                                       uint16_t* h_out, void* workspace, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* Q4_H */

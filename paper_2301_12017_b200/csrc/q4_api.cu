// q4_api.cu -- the C ABI (include/q4.h): argument validation, error reporting, kernel
// dispatch, and the host-side orchestration of the encoder layer / stack (a8).
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/q4.h"
#include "kernels.h"

namespace q4 {
static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
}  // namespace q4

namespace {

thread_local char g_err[512] = "";

q4_status fail(q4_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}
q4_status cuda_fail(cudaError_t e, const char* where) {
  return fail(Q4_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}
bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }
bool al4(const void* p) { return ((uintptr_t)p & 3) == 0; }
bool al8(const void* p) { return ((uintptr_t)p & 7) == 0; }

bool clip_ok(float c) {
  if (c == 0.f) return true;
  if (!(c > 0.f)) return false;
  __half h = __float2half_rn(c);
  return __half2float(h) == c;
}
size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

extern "C" {

const char* q4_last_error(void) { return g_err; }
const char* q4_version(void) { return "q4-b200 0.1 (sm_100a; tcgen05 kind::i8 W4A4)"; }
uint64_t q4_launch_count(void) { return q4::g_launches.load(); }

q4_status q4_launch_floor(int32_t n, int32_t ctas, void* stream) {
  g_err[0] = 0;
  if (n < 0 || n > 4096 || ctas < 1 || ctas > 1024)
    return fail(Q4_EINVAL, "q4_launch_floor: n=%d ctas=%d (need 0..4096, 1..1024)", n, ctas);
  for (int i = 0; i < n; ++i) {
    cudaError_t e = q4::launch_floor_kernel(ctas, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "q4_launch_floor");
  }
  return Q4_OK;
}

q4_status q4_quantize_rows(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x, float clip,
                           uint8_t* codes, float* scales, void* stream) {
  g_err[0] = 0;
  if (rows < 0 || cols <= 0 || ld_x < cols)
    return fail(Q4_ESHAPE, "q4_quantize_rows: rows=%lld cols=%lld ld_x=%lld (need rows>=0, cols>0, ld_x>=cols)",
                (long long)rows, (long long)cols, (long long)ld_x);
  if (cols % 8 || ld_x % 8)
    return fail(Q4_ESHAPE, "q4_quantize_rows: cols=%lld and ld_x=%lld must be multiples of 8",
                (long long)cols, (long long)ld_x);
  if (cols > (1 << 30)) return fail(Q4_ESHAPE, "q4_quantize_rows: cols=%lld too large", (long long)cols);
  if (rows == 0) return Q4_OK;
  if (!x || !codes || !scales) return fail(Q4_EINVAL, "q4_quantize_rows: NULL x/codes/scales");
  if (!al16(x) || !al4(codes) || !al4(scales))
    return fail(Q4_EALIGN, "q4_quantize_rows: x must be 16-byte aligned, codes/scales 4-byte aligned");
  if (!clip_ok(clip)) return fail(Q4_EINVAL, "q4_quantize_rows: clip=%g is not 0 or a positive fp16 value", clip);
  cudaError_t e = q4::launch_quantize_rows(reinterpret_cast<const __half*>(x), rows, (int)cols, ld_x, clip,
                                           codes, scales, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_quantize_rows");
}

q4_status q4_quantize_rows_i8(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x, float clip,
                              int8_t* codes, float* scales, void* stream) {
  g_err[0] = 0;
  if (rows < 0 || cols <= 0 || ld_x < cols)
    return fail(Q4_ESHAPE, "q4_quantize_rows_i8: rows=%lld cols=%lld ld_x=%lld (need rows>=0, cols>0, ld_x>=cols)",
                (long long)rows, (long long)cols, (long long)ld_x);
  if (cols % 8 || ld_x % 8)
    return fail(Q4_ESHAPE, "q4_quantize_rows_i8: cols=%lld and ld_x=%lld must be multiples of 8",
                (long long)cols, (long long)ld_x);
  if (cols > (1 << 30)) return fail(Q4_ESHAPE, "q4_quantize_rows_i8: cols=%lld too large", (long long)cols);
  if (rows == 0) return Q4_OK;
  if (!x || !codes || !scales) return fail(Q4_EINVAL, "q4_quantize_rows_i8: NULL x/codes/scales");
  if (!al16(x) || !al8(codes) || !al4(scales))
    return fail(Q4_EALIGN, "q4_quantize_rows_i8: x must be 16-byte aligned, codes 8-byte, scales 4-byte");
  if (!clip_ok(clip)) return fail(Q4_EINVAL, "q4_quantize_rows_i8: clip=%g is not 0 or a positive fp16 value", clip);
  cudaError_t e = q4::launch_quantize_rows_i8(reinterpret_cast<const __half*>(x), rows, (int)cols, ld_x, clip,
                                              codes, scales, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_quantize_rows_i8");
}

size_t q4_w8a8_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t kind) {
  return q4_w4a4_linear_workspace(M, N, K, kind);
}

q4_status q4_w8a8_linear(const int8_t* a_codes, const float* a_scales, const int8_t* w_codes,
                         const float* w_scales, int64_t M, int64_t N, int64_t K, const q4_epilogue* epi,
                         void* workspace, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!epi) return fail(Q4_EINVAL, "q4_w8a8_linear: epi is NULL");
  if (M < 0 || N <= 0 || K <= 0 || M > (1ll << 31) - 1 || N > (1 << 24))
    return fail(Q4_ESHAPE, "q4_w8a8_linear: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
  if (N % 32) return fail(Q4_ESHAPE, "q4_w8a8_linear: N=%lld must be a multiple of 32", (long long)N);
  if (K % 128) return fail(Q4_ESHAPE, "q4_w8a8_linear: K=%lld must be a multiple of 128 (one TMA k-block)", (long long)K);
  if (K > 131072) return fail(Q4_ESHAPE, "q4_w8a8_linear: K=%lld > 131072 would break the INT32 accumulator bound", (long long)K);
  const int kind = epi->kind;
  if (kind < Q4_EPI_I32 || kind > Q4_EPI_RESLN_Q4) return fail(Q4_EINVAL, "q4_w8a8_linear: unknown epilogue kind %d", kind);
  if (epi->mainloop != Q4_MAINLOOP_AUTO && epi->mainloop != Q4_MAINLOOP_TCGEN05)
    return fail(Q4_EUNSUPPORTED, "q4_w8a8_linear: mainloop %d (W8A8 runs on tcgen05 only)", epi->mainloop);
  if (M == 0) return Q4_OK;
  if (!a_codes || !a_scales || !w_codes || !w_scales)
    return fail(Q4_EINVAL, "q4_w8a8_linear: NULL operand (a_codes/a_scales/w_codes/w_scales)");
  if (!al16(a_codes) || !al16(w_codes) || !al4(a_scales) || !al16(w_scales))
    return fail(Q4_EALIGN, "q4_w8a8_linear: codes and w_scales must be 16-byte aligned, a_scales 4-byte aligned");
  if ((epi->bias && !al4(epi->bias)) || (epi->gamma && !al4(epi->gamma)) || (epi->beta && !al4(epi->beta)))
    return fail(Q4_EALIGN, "q4_w8a8_linear: bias/gamma/beta must be 4-byte aligned");
  switch (kind) {
    case Q4_EPI_I32:
      if (!epi->out_i32 || !al16(epi->out_i32)) return fail(Q4_EINVAL, "q4_w8a8_linear(I32): out_i32 NULL or not 16-byte aligned");
      break;
    case Q4_EPI_F16:
      if (!epi->out_f16 || !al16(epi->out_f16)) return fail(Q4_EINVAL, "q4_w8a8_linear(F16): out_f16 NULL or not 16-byte aligned");
      break;
    case Q4_EPI_GELU_Q4:
      if (!epi->out_codes || !epi->out_scales) return fail(Q4_EINVAL, "q4_w8a8_linear(GELU_Q): out_codes/out_scales NULL");
      if (!al16(epi->out_codes) || (epi->out_f16 && !al16(epi->out_f16)))
        return fail(Q4_EALIGN, "q4_w8a8_linear(GELU_Q): outputs must be 16-byte aligned");
      break;
    case Q4_EPI_RESLN_Q4:
      if (!epi->out_codes || !epi->out_scales || !epi->out_f16 || !epi->residual || !epi->gamma || !epi->beta)
        return fail(Q4_EINVAL, "q4_w8a8_linear(RESLN_Q): out_f16/out_codes/out_scales/residual/gamma/beta must be non-NULL");
      if (!al16(epi->out_codes) || !al16(epi->out_f16) || !al16(epi->residual))
        return fail(Q4_EALIGN, "q4_w8a8_linear(RESLN_Q): out_f16/out_codes/residual must be 16-byte aligned");
      if (!(epi->ln_eps >= 0.f)) return fail(Q4_EINVAL, "q4_w8a8_linear(RESLN_Q): ln_eps=%g", epi->ln_eps);
      break;
  }
  if (!clip_ok(epi->requant_clip)) return fail(Q4_EINVAL, "q4_w8a8_linear: requant_clip=%g is not 0 or a positive fp16 value", epi->requant_clip);
  if (kind == Q4_EPI_GELU_Q4 || kind == Q4_EPI_RESLN_Q4) {
    if (N % 64) return fail(Q4_ESHAPE, "q4_w8a8_linear: N=%lld must be a multiple of 64 for row epilogues", (long long)N);
    const size_t need = q4_w8a8_linear_workspace(M, N, K, kind);
    if (!workspace || ws_bytes < need)
      return fail(Q4_EINVAL, "q4_w8a8_linear: workspace %zu bytes < required %zu (q4_w8a8_linear_workspace)", ws_bytes, need);
    if (!al16(workspace)) return fail(Q4_EALIGN, "q4_w8a8_linear: workspace must be 16-byte aligned");
  }
  q4::GemmArgs g;
  g.a_codes = nullptr; g.a_i8 = a_codes; g.a_scales = a_scales; g.w_codes = nullptr; g.w_i8 = w_codes;
  g.w_scales = w_scales;
  g.M = (int)M; g.N = (int)N; g.K = (int)K; g.kind = kind; g.mainloop = Q4_MAINLOOP_TCGEN05;
  g.bias = reinterpret_cast<const __half*>(epi->bias);
  g.residual = reinterpret_cast<const __half*>(epi->residual);
  g.gamma = reinterpret_cast<const __half*>(epi->gamma);
  g.beta = reinterpret_cast<const __half*>(epi->beta);
  g.ln_eps = epi->ln_eps; g.clip = epi->requant_clip;
  g.out_i32 = epi->out_i32; g.out_f16 = reinterpret_cast<__half*>(epi->out_f16);
  g.out_codes = epi->out_codes; g.out_scales = epi->out_scales;
  const char* why = "";
  cudaError_t e = q4::launch_w4a4_tc(g, workspace, ws_bytes, (cudaStream_t)stream, &why);
  if (e == cudaErrorNotSupported) return fail(Q4_EUNSUPPORTED, "q4_w8a8_linear: %s (M=%lld N=%lld K=%lld)", why, (long long)M, (long long)N, (long long)K);
  if (e != cudaSuccess) return fail(Q4_ECUDA, "q4_w8a8_linear: %s %s", cudaGetErrorString(e), why);
  return Q4_OK;
}

q4_status q4_quantize_rows_asym(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld_x, uint8_t* codes,
                                float* scales, float* zeros, void* stream) {
  g_err[0] = 0;
  if (rows < 0 || cols <= 0 || ld_x < cols)
    return fail(Q4_ESHAPE, "q4_quantize_rows_asym: rows=%lld cols=%lld ld_x=%lld", (long long)rows, (long long)cols,
                (long long)ld_x);
  if (cols % 8 || ld_x % 8 || cols > 4096)
    return fail(Q4_ESHAPE, "q4_quantize_rows_asym: cols=%lld / ld_x=%lld (multiples of 8, cols <= 4096)",
                (long long)cols, (long long)ld_x);
  if (rows == 0) return Q4_OK;
  if (!x || !codes || !scales || !zeros) return fail(Q4_EINVAL, "q4_quantize_rows_asym: NULL x/codes/scales/zeros");
  if (!al16(x) || !al4(codes) || !al4(scales) || !al4(zeros))
    return fail(Q4_EALIGN, "q4_quantize_rows_asym: x 16-byte aligned, codes/scales/zeros 4-byte aligned");
  cudaError_t e = q4::launch_quantize_rows_asym(reinterpret_cast<const __half*>(x), rows, (int)cols, ld_x, codes,
                                                scales, zeros, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_quantize_rows_asym");
}

q4_status q4_weight_code_sums(const uint8_t* w_codes, int64_t N, int64_t K, float* sums, void* stream) {
  g_err[0] = 0;
  if (N < 0 || K <= 0 || K % 2) return fail(Q4_ESHAPE, "q4_weight_code_sums: N=%lld K=%lld", (long long)N, (long long)K);
  if (N == 0) return Q4_OK;
  if (!w_codes || !sums) return fail(Q4_EINVAL, "q4_weight_code_sums: NULL w_codes/sums");
  cudaError_t e = q4::launch_weight_code_sums(w_codes, N, K, sums, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_weight_code_sums");
}

q4_status q4_w4a4_asym_linear(const uint8_t* a_codes, const float* a_scales, const float* a_zeros,
                              const uint8_t* w_codes, const float* w_scales, const float* w_sums, int64_t M, int64_t N,
                              int64_t K, const q4_epilogue* epi, void* workspace, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!epi) return fail(Q4_EINVAL, "q4_w4a4_asym_linear: epi is NULL");
  const int kind = epi->kind;
  if (kind < Q4_EPI_I32 || kind > Q4_EPI_RESLN_Q4) return fail(Q4_EINVAL, "q4_w4a4_asym_linear: unknown epilogue kind %d", kind);
  if (epi->mainloop != Q4_MAINLOOP_AUTO && epi->mainloop != Q4_MAINLOOP_TCGEN05 && epi->mainloop != Q4_MAINLOOP_TCGEN05_W8)
    return fail(Q4_EUNSUPPORTED, "q4_w4a4_asym_linear: mainloop %d (tcgen05 only)", epi->mainloop);
  if (!a_zeros || (kind != Q4_EPI_I32 && !w_sums))
    return fail(Q4_EINVAL, "q4_w4a4_asym_linear: NULL a_zeros / w_sums");
  if (kind != Q4_EPI_I32 && !al16(w_sums)) return fail(Q4_EALIGN, "q4_w4a4_asym_linear: w_sums 16-byte aligned");
  // the validation of q4_w4a4_linear with the asymmetric fields set
  if (M < 0 || N <= 0 || K <= 0 || M > (1ll << 31) - 1 || N > (1 << 24) || N % 32 || K % 32 || K > 8192)
    return fail(Q4_ESHAPE, "q4_w4a4_asym_linear: M=%lld N=%lld K=%lld (N %% 32 == 0, K %% 32 == 0, K <= 8192)",
                (long long)M, (long long)N, (long long)K);
  if (M == 0) return Q4_OK;
  if (!a_codes || !a_scales || !w_codes || !w_scales)
    return fail(Q4_EINVAL, "q4_w4a4_asym_linear: NULL operand (a_codes/a_scales/w_codes/w_scales)");
  if (!al16(a_codes) || !al16(w_codes) || !al16(w_scales) || !al4(a_scales) || !al4(a_zeros))
    return fail(Q4_EALIGN, "q4_w4a4_asym_linear: codes / w_scales 16-byte aligned, a_scales / a_zeros 4-byte aligned");
  if ((epi->bias && !al4(epi->bias)) || (epi->gamma && !al4(epi->gamma)) || (epi->beta && !al4(epi->beta)))
    return fail(Q4_EALIGN, "q4_w4a4_asym_linear: bias/gamma/beta must be 4-byte aligned");
  if (epi->mainloop == Q4_MAINLOOP_TCGEN05_W8 && (!epi->w_i8 || !al16(epi->w_i8)))
    return fail(Q4_EINVAL, "q4_w4a4_asym_linear: TCGEN05_W8 needs 16-byte aligned epi->w_i8 (q4_prepack_weights)");
  if (epi->mainloop == Q4_MAINLOOP_AUTO && epi->w_i8 && !al16(epi->w_i8))
    return fail(Q4_EALIGN, "q4_w4a4_asym_linear: epi->w_i8 must be 16-byte aligned");
  switch (kind) {
    case Q4_EPI_I32:
      if (!epi->out_i32 || !al16(epi->out_i32)) return fail(Q4_EINVAL, "q4_w4a4_asym_linear(I32): out_i32 NULL or not 16-byte aligned");
      break;
    case Q4_EPI_F16:
      if (!epi->out_f16 || !al16(epi->out_f16)) return fail(Q4_EINVAL, "q4_w4a4_asym_linear(F16): out_f16 NULL or not 16-byte aligned");
      break;
    case Q4_EPI_GELU_Q4:
      if (!epi->out_codes || !epi->out_scales) return fail(Q4_EINVAL, "q4_w4a4_asym_linear(GELU_Q4): out_codes/out_scales NULL");
      if (!al16(epi->out_codes) || (epi->out_f16 && !al16(epi->out_f16)))
        return fail(Q4_EALIGN, "q4_w4a4_asym_linear(GELU_Q4): outputs must be 16-byte aligned");
      break;
    case Q4_EPI_RESLN_Q4:
      if (!epi->out_codes || !epi->out_scales || !epi->out_f16 || !epi->residual || !epi->gamma || !epi->beta)
        return fail(Q4_EINVAL, "q4_w4a4_asym_linear(RESLN_Q4): out_f16/out_codes/out_scales/residual/gamma/beta must be non-NULL");
      if (!al16(epi->out_codes) || !al16(epi->out_f16) || !al16(epi->residual))
        return fail(Q4_EALIGN, "q4_w4a4_asym_linear(RESLN_Q4): out_f16/out_codes/residual must be 16-byte aligned");
      if (!(epi->ln_eps >= 0.f)) return fail(Q4_EINVAL, "q4_w4a4_asym_linear(RESLN_Q4): ln_eps=%g", epi->ln_eps);
      break;
  }
  if (epi->requant_clip != 0.f) return fail(Q4_EUNSUPPORTED, "q4_w4a4_asym_linear: requant_clip must be 0");
  if (kind == Q4_EPI_GELU_Q4 || kind == Q4_EPI_RESLN_Q4) {
    if (N % 64) return fail(Q4_ESHAPE, "q4_w4a4_asym_linear: N=%lld must be a multiple of 64 for row epilogues", (long long)N);
    if (epi->out_zeros && !al4(epi->out_zeros)) return fail(Q4_EALIGN, "q4_w4a4_asym_linear: out_zeros 4-byte aligned");
    const size_t need = q4_w4a4_linear_workspace(M, N, K, kind);
    if (!workspace || ws_bytes < need)
      return fail(Q4_EINVAL, "q4_w4a4_asym_linear: workspace %zu bytes < required %zu (q4_w4a4_linear_workspace)", ws_bytes, need);
    if (!al16(workspace)) return fail(Q4_EALIGN, "q4_w4a4_asym_linear: workspace must be 16-byte aligned");
  }
  q4::GemmArgs g;
  g.a_codes = a_codes; g.a_i8 = nullptr; g.a_scales = a_scales; g.w_codes = w_codes; g.w_scales = w_scales;
  g.a_zeros = a_zeros; g.w_sums = w_sums;
  g.M = (int)M; g.N = (int)N; g.K = (int)K; g.kind = kind; g.mainloop = epi->mainloop;
  g.bias = reinterpret_cast<const __half*>(epi->bias);
  g.residual = reinterpret_cast<const __half*>(epi->residual);
  g.gamma = reinterpret_cast<const __half*>(epi->gamma);
  g.beta = reinterpret_cast<const __half*>(epi->beta);
  g.ln_eps = epi->ln_eps; g.clip = 0.f;
  g.out_i32 = epi->out_i32; g.out_f16 = reinterpret_cast<__half*>(epi->out_f16); g.out_codes = epi->out_codes;
  g.out_scales = epi->out_scales;
  g.out_zeros = (kind == Q4_EPI_GELU_Q4 || kind == Q4_EPI_RESLN_Q4) ? epi->out_zeros : nullptr;
  g.w_i8 = (epi->mainloop != Q4_MAINLOOP_TCGEN05 && epi->w_i8) ? epi->w_i8 : nullptr;
  const char* why = "";
  cudaError_t e = q4::launch_w4a4_tc(g, workspace, ws_bytes, (cudaStream_t)stream, &why);
  if (e == cudaErrorNotSupported) return fail(Q4_EUNSUPPORTED, "q4_w4a4_asym_linear: %s", why);
  if (e != cudaSuccess) return fail(Q4_ECUDA, "q4_w4a4_asym_linear: %s %s", cudaGetErrorString(e), why);
  return Q4_OK;
}

size_t q4_f16_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t kind) {
  return q4_w4a4_linear_workspace(M, N, K, kind);
}

q4_status q4_f16_linear(const uint16_t* a, const uint16_t* w, int64_t M, int64_t N, int64_t K, const q4_epilogue* epi,
                        void* workspace, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!epi) return fail(Q4_EINVAL, "q4_f16_linear: epi is NULL");
  if (M < 0 || N <= 0 || K <= 0 || M > (1ll << 31) - 1 || N > (1 << 24) || K > (1 << 20))
    return fail(Q4_ESHAPE, "q4_f16_linear: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
  if (N % 32) return fail(Q4_ESHAPE, "q4_f16_linear: N=%lld must be a multiple of 32", (long long)N);
  if (K % 64) return fail(Q4_ESHAPE, "q4_f16_linear: K=%lld must be a multiple of 64 (one 128-byte k-block)", (long long)K);
  const int kind = epi->kind;
  if (kind != Q4_EPI_F16 && kind != Q4_EPI_GELU_Q4 && kind != Q4_EPI_RESLN_Q4)
    return fail(Q4_EINVAL, "q4_f16_linear: epilogue kind %d (F16, GELU_Q4 or RESLN_Q4)", kind);
  if (epi->mainloop != Q4_MAINLOOP_AUTO && epi->mainloop != Q4_MAINLOOP_TCGEN05)
    return fail(Q4_EUNSUPPORTED, "q4_f16_linear: mainloop %d (tcgen05 only)", epi->mainloop);
  if (M == 0) return Q4_OK;
  if (!a || !w) return fail(Q4_EINVAL, "q4_f16_linear: NULL a/w");
  if (!al16(a) || !al16(w)) return fail(Q4_EALIGN, "q4_f16_linear: a and w must be 16-byte aligned");
  if ((epi->bias && !al4(epi->bias)) || (epi->gamma && !al4(epi->gamma)) || (epi->beta && !al4(epi->beta)))
    return fail(Q4_EALIGN, "q4_f16_linear: bias/gamma/beta must be 4-byte aligned");
  if (kind == Q4_EPI_F16 && (!epi->out_f16 || !al16(epi->out_f16)))
    return fail(Q4_EINVAL, "q4_f16_linear(F16): out_f16 NULL or not 16-byte aligned");
  if (kind == Q4_EPI_GELU_Q4) {
    if (!epi->out_codes || !epi->out_scales) return fail(Q4_EINVAL, "q4_f16_linear(GELU_Q4): out_codes/out_scales NULL");
    if (!al16(epi->out_codes) || (epi->out_f16 && !al16(epi->out_f16)))
      return fail(Q4_EALIGN, "q4_f16_linear(GELU_Q4): outputs must be 16-byte aligned");
  }
  if (kind == Q4_EPI_RESLN_Q4) {
    if (!epi->out_codes || !epi->out_scales || !epi->out_f16 || !epi->residual || !epi->gamma || !epi->beta)
      return fail(Q4_EINVAL, "q4_f16_linear(RESLN_Q4): out_f16/out_codes/out_scales/residual/gamma/beta must be non-NULL");
    if (!al16(epi->out_codes) || !al16(epi->out_f16) || !al16(epi->residual))
      return fail(Q4_EALIGN, "q4_f16_linear(RESLN_Q4): out_f16/out_codes/residual must be 16-byte aligned");
    if (!(epi->ln_eps >= 0.f)) return fail(Q4_EINVAL, "q4_f16_linear(RESLN_Q4): ln_eps=%g", epi->ln_eps);
  }
  if (!clip_ok(epi->requant_clip)) return fail(Q4_EINVAL, "q4_f16_linear: requant_clip=%g is not 0 or a positive fp16 value", epi->requant_clip);
  if (kind == Q4_EPI_GELU_Q4 || kind == Q4_EPI_RESLN_Q4) {
    if (N % 64) return fail(Q4_ESHAPE, "q4_f16_linear: N=%lld must be a multiple of 64 for row epilogues", (long long)N);
    const size_t need = q4_f16_linear_workspace(M, N, K, kind);
    if (!workspace || ws_bytes < need)
      return fail(Q4_EINVAL, "q4_f16_linear: workspace %zu bytes < required %zu (q4_f16_linear_workspace)", ws_bytes, need);
    if (!al16(workspace)) return fail(Q4_EALIGN, "q4_f16_linear: workspace must be 16-byte aligned");
  }
  q4::GemmArgs g;
  g.a_codes = nullptr; g.a_i8 = reinterpret_cast<const int8_t*>(a); g.a_scales = nullptr;
  g.w_codes = nullptr; g.w_i8 = reinterpret_cast<const int8_t*>(w); g.w_scales = nullptr;
  g.f16_ops = true;
  g.M = (int)M; g.N = (int)N; g.K = (int)(2 * K); g.kind = kind; g.mainloop = Q4_MAINLOOP_TCGEN05;
  g.bias = reinterpret_cast<const __half*>(epi->bias);
  g.residual = reinterpret_cast<const __half*>(epi->residual);
  g.gamma = reinterpret_cast<const __half*>(epi->gamma);
  g.beta = reinterpret_cast<const __half*>(epi->beta);
  g.ln_eps = epi->ln_eps; g.clip = epi->requant_clip;
  g.out_i32 = nullptr; g.out_f16 = reinterpret_cast<__half*>(epi->out_f16);
  g.out_codes = epi->out_codes; g.out_scales = epi->out_scales;
  const char* why = "";
  cudaError_t e = q4::launch_w4a4_tc(g, workspace, ws_bytes, (cudaStream_t)stream, &why);
  if (e == cudaErrorNotSupported) return fail(Q4_EUNSUPPORTED, "q4_f16_linear: %s (M=%lld N=%lld K=%lld)", why, (long long)M, (long long)N, (long long)K);
  if (e != cudaSuccess) return fail(Q4_ECUDA, "q4_f16_linear: %s %s", cudaGetErrorString(e), why);
  return Q4_OK;
}

size_t q4_w4a4_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t kind) {
  (void)K;
  if (kind != Q4_EPI_GELU_Q4 && kind != Q4_EPI_RESLN_Q4 && kind != Q4_EPI_F16 && kind != Q4_EPI_I32) return 0;
  if (M <= 0 || N <= 0 || M > (1ll << 31) - 1 || N > (1 << 24)) return 0;
  return q4::tc_workspace_bytes((int)M, (int)N, q4::tc_tile_n((int)M, (int)N, kind), kind);
}

q4_status q4_w4a4_linear(const uint8_t* a_codes, const float* a_scales, const uint8_t* w_codes,
                         const float* w_scales, int64_t M, int64_t N, int64_t K, const q4_epilogue* epi,
                         void* workspace, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!epi) return fail(Q4_EINVAL, "q4_w4a4_linear: epi is NULL");
  if (M < 0 || N <= 0 || K <= 0 || M > (1ll << 31) - 1 || N > (1 << 24))
    return fail(Q4_ESHAPE, "q4_w4a4_linear: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
  if (N % 32) return fail(Q4_ESHAPE, "q4_w4a4_linear: N=%lld must be a multiple of 32", (long long)N);
  if (K % 32) return fail(Q4_ESHAPE, "q4_w4a4_linear: K=%lld must be a multiple of 32 (16-byte packed rows)", (long long)K);
  if (K > 8192) return fail(Q4_ESHAPE, "q4_w4a4_linear: K=%lld > 8192 would break the INT32 accumulator bound", (long long)K);
  const int kind = epi->kind;
  if (kind < Q4_EPI_I32 || kind > Q4_EPI_RESLN_Q4) return fail(Q4_EINVAL, "q4_w4a4_linear: unknown epilogue kind %d", kind);
  if (M == 0) return Q4_OK;
  if (!a_codes || !a_scales || !w_codes || !w_scales)
    return fail(Q4_EINVAL, "q4_w4a4_linear: NULL operand (a_codes/a_scales/w_codes/w_scales)");
  if (!al16(a_codes) || !al16(w_codes) || !al4(a_scales) || !al16(w_scales))
    return fail(Q4_EALIGN, "q4_w4a4_linear: codes and w_scales must be 16-byte aligned, a_scales 4-byte aligned");
  if ((epi->bias && !al4(epi->bias)) || (epi->gamma && !al4(epi->gamma)) || (epi->beta && !al4(epi->beta)))
    return fail(Q4_EALIGN, "q4_w4a4_linear: bias/gamma/beta must be 4-byte aligned");
  switch (kind) {
    case Q4_EPI_I32:
      if (!epi->out_i32 || !al16(epi->out_i32)) return fail(Q4_EINVAL, "q4_w4a4_linear(I32): out_i32 NULL or not 16-byte aligned");
      break;
    case Q4_EPI_F16:
      if (!epi->out_f16 || !al16(epi->out_f16)) return fail(Q4_EINVAL, "q4_w4a4_linear(F16): out_f16 NULL or not 16-byte aligned");
      break;
    case Q4_EPI_GELU_Q4:
      if (!epi->out_codes || !epi->out_scales) return fail(Q4_EINVAL, "q4_w4a4_linear(GELU_Q4): out_codes/out_scales NULL");
      if (!al16(epi->out_codes) || (epi->out_f16 && !al16(epi->out_f16)))
        return fail(Q4_EALIGN, "q4_w4a4_linear(GELU_Q4): outputs must be 16-byte aligned");
      break;
    case Q4_EPI_RESLN_Q4:
      if (!epi->out_codes || !epi->out_scales || !epi->out_f16 || !epi->residual || !epi->gamma || !epi->beta)
        return fail(Q4_EINVAL, "q4_w4a4_linear(RESLN_Q4): out_f16/out_codes/out_scales/residual/gamma/beta must be non-NULL");
      if (!al16(epi->out_codes) || !al16(epi->out_f16) || !al16(epi->residual))
        return fail(Q4_EALIGN, "q4_w4a4_linear(RESLN_Q4): out_f16/out_codes/residual must be 16-byte aligned");
      if (!(epi->ln_eps >= 0.f)) return fail(Q4_EINVAL, "q4_w4a4_linear(RESLN_Q4): ln_eps=%g", epi->ln_eps);
      break;
  }
  if (!clip_ok(epi->requant_clip)) return fail(Q4_EINVAL, "q4_w4a4_linear: requant_clip=%g is not 0 or a positive fp16 value", epi->requant_clip);
  if (kind == Q4_EPI_GELU_Q4 || kind == Q4_EPI_RESLN_Q4) {
    if (N % 64) return fail(Q4_ESHAPE, "q4_w4a4_linear: N=%lld must be a multiple of 64 for row epilogues", (long long)N);
    const size_t need = q4_w4a4_linear_workspace(M, N, K, kind);
    if (!workspace || ws_bytes < need)
      return fail(Q4_EINVAL, "q4_w4a4_linear: workspace %zu bytes < required %zu (q4_w4a4_linear_workspace)", ws_bytes, need);
    if (!al16(workspace)) return fail(Q4_EALIGN, "q4_w4a4_linear: workspace must be 16-byte aligned");
  }
  q4::GemmArgs g;
  g.a_codes = a_codes; g.a_i8 = nullptr; g.a_scales = a_scales; g.w_codes = w_codes; g.w_scales = w_scales;
  g.M = (int)M; g.N = (int)N; g.K = (int)K; g.kind = kind; g.mainloop = epi->mainloop;
  g.bias = reinterpret_cast<const __half*>(epi->bias);
  g.residual = reinterpret_cast<const __half*>(epi->residual);
  g.gamma = reinterpret_cast<const __half*>(epi->gamma);
  g.beta = reinterpret_cast<const __half*>(epi->beta);
  g.ln_eps = epi->ln_eps; g.clip = epi->requant_clip;
  g.out_i32 = epi->out_i32; g.out_f16 = reinterpret_cast<__half*>(epi->out_f16);
  g.out_codes = epi->out_codes; g.out_scales = epi->out_scales;
  g.out_zeros = (kind == Q4_EPI_GELU_Q4 || kind == Q4_EPI_RESLN_Q4) ? epi->out_zeros : nullptr;
  if (g.out_zeros && (epi->requant_clip != 0.f || !al4(g.out_zeros)))
    return fail(Q4_EUNSUPPORTED, "q4_w4a4_linear: asymmetric requant (out_zeros) needs requant_clip 0 and 4-byte aligned zeros");
  if (g.out_zeros && (epi->mainloop == Q4_MAINLOOP_MMA_SYNC_S8 || epi->mainloop == Q4_MAINLOOP_MMA_SYNC_S4))
    return fail(Q4_EUNSUPPORTED, "q4_w4a4_linear: asymmetric requant on the tcgen05 mainloops only");
  g.w_i8 = nullptr;
  if (epi->mainloop == Q4_MAINLOOP_TCGEN05_W8 || epi->mainloop == Q4_MAINLOOP_TCGEN05_W8_1CTA ||
      (epi->mainloop == Q4_MAINLOOP_AUTO && epi->w_i8)) {
    if (!epi->w_i8 || !al16(epi->w_i8))
      return fail(Q4_EINVAL, "q4_w4a4_linear: TCGEN05_W8 needs 16-byte aligned epi->w_i8 (q4_prepack_weights)");
    g.w_i8 = epi->w_i8;
  }
  const char* why = "";
  cudaError_t e;
  switch (epi->mainloop) {
    case Q4_MAINLOOP_AUTO:
    case Q4_MAINLOOP_TCGEN05:
    case Q4_MAINLOOP_TCGEN05_W8:
    case Q4_MAINLOOP_TCGEN05_W8_1CTA: e = q4::launch_w4a4_tc(g, workspace, ws_bytes, (cudaStream_t)stream, &why); break;
    case Q4_MAINLOOP_MMA_SYNC_S8: e = q4::launch_w4a4_legacy(g, false, (cudaStream_t)stream, &why); break;
    case Q4_MAINLOOP_MMA_SYNC_S4: e = q4::launch_w4a4_legacy(g, true, (cudaStream_t)stream, &why); break;
    default: return fail(Q4_EINVAL, "q4_w4a4_linear: unknown mainloop %d", epi->mainloop);
  }
  if (e == cudaErrorNotSupported) return fail(Q4_EUNSUPPORTED, "q4_w4a4_linear: %s (M=%lld N=%lld K=%lld)", why, (long long)M, (long long)N, (long long)K);
  if (e != cudaSuccess) return fail(Q4_ECUDA, "q4_w4a4_linear: %s %s", cudaGetErrorString(e), why);
  return Q4_OK;
}

// ------------------------------------------------------------------ NEXT-4: 2:4-sparse weights

q4_status q4_prune_24(const uint16_t* w, int64_t N, int64_t K, uint16_t* out, void* stream) {
  g_err[0] = 0;
  if (N < 0 || K <= 0 || K % 4) return fail(Q4_ESHAPE, "q4_prune_24: N=%lld K=%lld (K %% 4 == 0)", (long long)N, (long long)K);
  if (N == 0) return Q4_OK;
  if (!w || !out) return fail(Q4_EINVAL, "q4_prune_24: NULL w/out");
  if (!al8(w) || !al8(out)) return fail(Q4_EALIGN, "q4_prune_24: w/out must be 8-byte aligned");
  cudaError_t e = q4::launch_prune24(reinterpret_cast<const __half*>(w), N, K, reinterpret_cast<__half*>(out),
                                     (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_prune_24");
}

q4_status q4_sparse24_compress(const uint8_t* w_codes, int64_t N, int64_t K, int8_t* w_vals, uint32_t* w_meta,
                               int32_t* violations, void* stream) {
  g_err[0] = 0;
  if (N < 0 || K <= 0 || K % 256) return fail(Q4_ESHAPE, "q4_sparse24_compress: N=%lld K=%lld (K %% 256 == 0)", (long long)N, (long long)K);
  if (N == 0) return Q4_OK;
  if (!w_codes || !w_vals || !w_meta) return fail(Q4_EINVAL, "q4_sparse24_compress: NULL w_codes/w_vals/w_meta");
  if (!al16(w_codes) || !al16(w_vals) || !al16(w_meta) || (violations && !al4(violations)))
    return fail(Q4_EALIGN, "q4_sparse24_compress: pointers must be 16-byte aligned (violations 4)");
  cudaError_t e = q4::launch_sparse24_compress(w_codes, N, K, w_vals, w_meta, violations, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_sparse24_compress");
}

q4_status q4_w4a4_sparse24_linear(const uint8_t* a_codes, const float* a_scales, const int8_t* w_vals,
                                  const uint32_t* w_meta, const float* w_scales, int64_t M, int64_t N, int64_t K,
                                  const q4_epilogue* epi, void* stream) {
  g_err[0] = 0;
  if (!epi) return fail(Q4_EINVAL, "q4_w4a4_sparse24_linear: epi is NULL");
  if (epi->kind != Q4_EPI_F16 && epi->kind != Q4_EPI_I32)
    return fail(Q4_EUNSUPPORTED, "q4_w4a4_sparse24_linear: epilogue kind %d (F16 or I32)", epi->kind);
  if (M < 0 || N <= 0 || K <= 0 || M > (1ll << 31) - 1 || N % 128 || K % 256 || K > 8192)
    return fail(Q4_ESHAPE, "q4_w4a4_sparse24_linear: M=%lld N=%lld K=%lld (N %% 128 == 0, K %% 256 == 0, K <= 8192)",
                (long long)M, (long long)N, (long long)K);
  if (M == 0) return Q4_OK;
  if (!a_codes || !a_scales || !w_vals || !w_meta || !w_scales)
    return fail(Q4_EINVAL, "q4_w4a4_sparse24_linear: NULL operand");
  if (!al16(a_codes) || !al16(w_vals) || !al16(w_meta) || !al4(w_scales) || !al4(a_scales) ||
      (epi->bias && !al4(epi->bias)))
    return fail(Q4_EALIGN, "q4_w4a4_sparse24_linear: codes / values / metadata 16-byte aligned, scales / bias 4-byte");
  if ((epi->kind == Q4_EPI_F16 && (!epi->out_f16 || !al16(epi->out_f16))) ||
      (epi->kind == Q4_EPI_I32 && (!epi->out_i32 || !al16(epi->out_i32))))
    return fail(Q4_EINVAL, "q4_w4a4_sparse24_linear: output NULL or not 16-byte aligned");
  q4::SparseArgs g;
  g.a_codes = a_codes; g.a_scales = a_scales; g.w_vals = w_vals; g.w_meta = w_meta; g.w_scales = w_scales;
  g.bias = reinterpret_cast<const __half*>(epi->bias);
  g.M = (int)M; g.N = (int)N; g.K = (int)K;
  g.out_i32 = epi->kind == Q4_EPI_I32 ? epi->out_i32 : nullptr;
  g.out_f16 = epi->kind == Q4_EPI_F16 ? reinterpret_cast<__half*>(epi->out_f16) : nullptr;
  const char* why = "";
  cudaError_t e = q4::launch_w4a4_sparse24(g, (cudaStream_t)stream, &why);
  if (e == cudaErrorNotSupported) return fail(Q4_EUNSUPPORTED, "q4_w4a4_sparse24_linear: %s", why);
  if (e != cudaSuccess) return fail(Q4_ECUDA, "q4_w4a4_sparse24_linear: %s %s", cudaGetErrorString(e), why);
  return Q4_OK;
}

q4_status q4_prepack_weights(const uint8_t* w_codes, int64_t N, int64_t K, int8_t* w_i8, void* stream) {
  g_err[0] = 0;
  if (N < 0 || K <= 0 || K % 32) return fail(Q4_ESHAPE, "q4_prepack_weights: N=%lld K=%lld (need K %% 32 == 0)", (long long)N, (long long)K);
  if (N == 0) return Q4_OK;
  if (!w_codes || !w_i8) return fail(Q4_EINVAL, "q4_prepack_weights: NULL w_codes/w_i8");
  if (!al16(w_codes) || !al16(w_i8)) return fail(Q4_EALIGN, "q4_prepack_weights: pointers must be 16-byte aligned");
  cudaError_t e = q4::launch_prepack_weights(w_codes, N, K, w_i8, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_prepack_weights");
}

q4_status q4_attention_f16_q4(const uint16_t* qkv, int64_t B, int64_t S, int32_t heads, int32_t head_dim,
                              uint16_t* ctx_f16, uint8_t* ctx_codes, float* ctx_scales, void* stream) {
  g_err[0] = 0;
  if (head_dim != 64) return fail(Q4_EUNSUPPORTED, "q4_attention_f16_q4: head_dim=%d (only 64)", head_dim);
  if (B < 0 || S < 1 || S > 128) return fail(Q4_ESHAPE, "q4_attention_f16_q4: B=%lld S=%lld (need B>=0, 1<=S<=128)", (long long)B, (long long)S);
  if (heads < 1 || heads * 64 > 1024) return fail(Q4_ESHAPE, "q4_attention_f16_q4: heads=%d (need 1..16)", heads);
  if (B > 65535) return fail(Q4_ESHAPE, "q4_attention_f16_q4: B=%lld > 65535", (long long)B);
  if (B == 0) return Q4_OK;
  if (!qkv || !ctx_f16 || !ctx_codes || !ctx_scales)
    return fail(Q4_EINVAL, "q4_attention_f16_q4: NULL qkv/ctx_f16/ctx_codes/ctx_scales");
  if (!al16(qkv) || !al4(ctx_codes) || !al16(ctx_f16))
    return fail(Q4_EALIGN, "q4_attention_f16_q4: qkv/ctx_f16 must be 16-byte aligned, codes 4-byte");
  const __half* q = reinterpret_cast<const __half*>(qkv);
  __half* cf = reinterpret_cast<__half*>(ctx_f16);
  cudaError_t e = q4::launch_attention_tc(q, (int)B, (int)S, heads, cf, ctx_codes, ctx_scales, (cudaStream_t)stream);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_attention_f16_q4");
}

q4_status q4_attention_f16_q4_asym(const uint16_t* qkv, int64_t B, int64_t S, int32_t heads, int32_t head_dim,
                                   uint16_t* ctx_f16, uint8_t* ctx_codes, float* ctx_scales, float* ctx_zeros,
                                   void* stream) {
  g_err[0] = 0;
  if (head_dim != 64) return fail(Q4_EUNSUPPORTED, "q4_attention_f16_q4_asym: head_dim=%d (only 64)", head_dim);
  if (B < 0 || S < 1 || S > 128) return fail(Q4_ESHAPE, "q4_attention_f16_q4_asym: B=%lld S=%lld (need B>=0, 1<=S<=128)", (long long)B, (long long)S);
  if (heads < 1 || heads * 64 > 1024) return fail(Q4_ESHAPE, "q4_attention_f16_q4_asym: heads=%d (need 1..16)", heads);
  if (B > 65535) return fail(Q4_ESHAPE, "q4_attention_f16_q4_asym: B=%lld > 65535", (long long)B);
  if (B == 0) return Q4_OK;
  if (!qkv || !ctx_f16 || !ctx_codes || !ctx_scales || !ctx_zeros)
    return fail(Q4_EINVAL, "q4_attention_f16_q4_asym: NULL qkv/ctx_f16/ctx_codes/ctx_scales/ctx_zeros");
  if (!al16(qkv) || !al4(ctx_codes) || !al16(ctx_f16) || !al4(ctx_zeros))
    return fail(Q4_EALIGN, "q4_attention_f16_q4_asym: qkv/ctx_f16 16-byte aligned, codes / zeros 4-byte");
  cudaError_t e = q4::launch_attention_tc(reinterpret_cast<const __half*>(qkv), (int)B, (int)S, heads,
                                          reinterpret_cast<__half*>(ctx_f16), ctx_codes, ctx_scales,
                                          (cudaStream_t)stream, false, ctx_zeros);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_attention_f16_q4_asym");
}

q4_status q4_attention_f16_q8(const uint16_t* qkv, int64_t B, int64_t S, int32_t heads, int32_t head_dim,
                              uint16_t* ctx_f16, int8_t* ctx_codes, float* ctx_scales, void* stream) {
  g_err[0] = 0;
  if (head_dim != 64) return fail(Q4_EUNSUPPORTED, "q4_attention_f16_q8: head_dim=%d (only 64)", head_dim);
  if (B < 0 || S < 1 || S > 128) return fail(Q4_ESHAPE, "q4_attention_f16_q8: B=%lld S=%lld (need B>=0, 1<=S<=128)", (long long)B, (long long)S);
  if (heads < 1 || heads * 64 > 1024) return fail(Q4_ESHAPE, "q4_attention_f16_q8: heads=%d (need 1..16)", heads);
  if (B > 65535) return fail(Q4_ESHAPE, "q4_attention_f16_q8: B=%lld > 65535", (long long)B);
  if (B == 0) return Q4_OK;
  if (!qkv || !ctx_f16 || !ctx_codes || !ctx_scales)
    return fail(Q4_EINVAL, "q4_attention_f16_q8: NULL qkv/ctx_f16/ctx_codes/ctx_scales");
  if (!al16(qkv) || !al8(ctx_codes) || !al16(ctx_f16))
    return fail(Q4_EALIGN, "q4_attention_f16_q8: qkv/ctx_f16 must be 16-byte aligned, codes 8-byte");
  cudaError_t e = q4::launch_attention_tc(reinterpret_cast<const __half*>(qkv), (int)B, (int)S, heads,
                                          reinterpret_cast<__half*>(ctx_f16), reinterpret_cast<uint8_t*>(ctx_codes),
                                          ctx_scales, (cudaStream_t)stream, true);
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_attention_f16_q8");
}

// ------------------------------------------------------------------ encoder layer

namespace {
struct LayerWs {
  uint8_t* gemm_ws;
  size_t gemm_ws_bytes;
  uint16_t* qkv;
  uint16_t* ctx;
  uint8_t* ctx_codes;
  float* ctx_scales;
  uint16_t* h1;
  uint8_t* h1_codes;
  float* h1_scales;
  uint8_t* f_codes;
  float* f_scales;
  float *ctx_zeros, *h1_zeros, *f_zeros;  // asymmetric activations (cfg->asym_acts)
  uint16_t* ffn1;  // fp16 MLP intermediate, only when the MLP output part runs in FP16
  size_t bytes;
};
LayerWs layer_ws(const q4_layer_cfg* c, int64_t M, uint8_t* base, bool i8 = false) {
  LayerWs w;
  size_t o = 0;
  const int64_t h = c->hidden, f = c->ffn;
  const int64_t cd = i8 ? 1 : 2;  // elements per code byte
  auto take = [&](size_t n) { size_t r = o; o = align_up(o + n); return base ? base + r : nullptr; };
  size_t gw = 0;
  for (int64_t n : {h, f})
    for (int kind : {Q4_EPI_GELU_Q4, Q4_EPI_RESLN_Q4}) {
      size_t b = q4_w4a4_linear_workspace(M, n, 0, kind);
      if (b > gw) gw = b;
    }
  w.gemm_ws_bytes = gw;
  w.gemm_ws = take(gw);
  w.qkv = (uint16_t*)take((size_t)M * 3 * h * 2);
  w.ctx = (uint16_t*)take((size_t)M * h * 2);
  w.ctx_codes = take((size_t)(M * h / cd));
  w.ctx_scales = (float*)take((size_t)M * 4);
  w.h1 = (uint16_t*)take((size_t)M * h * 2);
  w.h1_codes = take((size_t)(M * h / cd));
  w.h1_scales = (float*)take((size_t)M * 4);
  w.f_codes = take((size_t)(M * f / cd));
  w.f_scales = (float*)take((size_t)M * 4);
  const bool az = !i8 && c->asym_acts;
  w.ctx_zeros = az ? (float*)take((size_t)M * 4) : nullptr;
  w.h1_zeros = az ? (float*)take((size_t)M * 4) : nullptr;
  w.f_zeros = az ? (float*)take((size_t)M * 4) : nullptr;
  w.ffn1 = (!i8 && (c->fp16_parts & 8)) ? (uint16_t*)take((size_t)M * f * 2) : nullptr;
  w.bytes = o;
  return w;
}
q4_status check_cfg(const q4_layer_cfg* c, const char* who) {
  if (!c) return fail(Q4_EINVAL, "%s: cfg is NULL", who);
  if (c->head_dim != 64 || c->heads < 1 || c->heads * 64 != c->hidden || c->hidden > 1024)
    return fail(Q4_EUNSUPPORTED, "%s: hidden=%d heads=%d head_dim=%d (need head_dim 64, hidden = 64*heads <= 1024)",
                who, c->hidden, c->heads, c->head_dim);
  if (c->ffn % 32 || c->ffn <= 0 || c->ffn > 4096) return fail(Q4_ESHAPE, "%s: ffn=%d (need multiple of 32, <= 4096)", who, c->ffn);
  if (c->fp16_parts < 0 || c->fp16_parts > 15) return fail(Q4_EINVAL, "%s: fp16_parts=%d (bits 0..3)", who, c->fp16_parts);
  if (c->asym_acts != 0 && c->asym_acts != 1) return fail(Q4_EINVAL, "%s: asym_acts=%d (0 or 1)", who, c->asym_acts);
  if (c->asym_acts && c->fp16_parts)
    return fail(Q4_EUNSUPPORTED, "%s: asym_acts with fp16_parts=%d (the asymmetric layer quantizes all four parts)", who,
                c->fp16_parts);
  return Q4_OK;
}
}  // namespace

size_t q4_encoder_layer_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S) {
  if (!cfg) return 0;
  return layer_ws(cfg, B * S, nullptr).bytes;
}

size_t q4_encoder_layer_w8a8_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S) {
  if (!cfg) return 0;
  return layer_ws(cfg, B * S, nullptr, true).bytes;
}

}  // extern "C"

namespace {
// One post-LN layer; i8 = the W8A8 baseline (int8 codes everywhere, q4_w8a8_linear and the
// int8 ctx quantize; the weight fields hold int8 codes [N, K], the *8 fields are unused).
q4_status encoder_layer_impl(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B, int64_t S,
                             const uint16_t* h_in, const uint8_t* hq_in, const float* hs_in, uint16_t* h_out,
                             uint8_t* hq_out, float* hs_out, void* workspace, size_t ws_bytes, const q4_taps* taps,
                             void* stream, bool i8, const float* hz_in = nullptr, float* hz_out = nullptr) {
  const char* who = i8 ? "q4_encoder_layer_w8a8" : (cfg && cfg->asym_acts) ? "q4_encoder_layer_asym" : "q4_encoder_layer";
  q4_status st = check_cfg(cfg, who);
  if (st) return st;
  if (!w) return fail(Q4_EINVAL, "%s: weights NULL", who);
  const bool asym = cfg->asym_acts != 0;
  if (i8 && asym) return fail(Q4_EUNSUPPORTED, "%s: asym_acts on the W8A8 baseline", who);
  if (asym && (!hz_in || !hz_out || !w->cqkv || !w->co || !w->c1 || !w->c2))
    return fail(Q4_EINVAL, "%s: asym_acts needs hz_in / hz_out and the weight code sums cqkv/co/c1/c2", who);
  if (B < 0 || S < 1 || S > 128) return fail(Q4_ESHAPE, "%s: B=%lld S=%lld", who, (long long)B, (long long)S);
  const int64_t M = B * S, h = cfg->hidden, f = cfg->ffn;
  if (M == 0) return Q4_OK;
  const int fp = cfg->fp16_parts;
  if (i8 && fp) return fail(Q4_EUNSUPPORTED, "%s: fp16_parts=%d (the W8A8 baseline quantizes all four parts)", who, fp);
  if (((fp & 1) && !w->fqkv) || ((fp & 2) && !w->fo) || ((fp & 4) && !w->f1) || ((fp & 8) && !w->f2))
    return fail(Q4_EINVAL, "%s: fp16_parts=%d needs the fp16 weights (fqkv/fo/f1/f2) of those parts", who, fp);
  LayerWs ws = layer_ws(cfg, M, (uint8_t*)workspace, i8);
  if (!workspace || ws_bytes < ws.bytes)
    return fail(Q4_EINVAL, "%s: workspace %zu bytes < required %zu", who, ws_bytes, ws.bytes);
  q4_taps tp;
  memset(&tp, 0, sizeof tp);
  if (taps) tp = *taps;
  // taps redirect the intermediates that have a tap buffer of the same layout
  uint16_t* qkv = tp.qkv ? tp.qkv : ws.qkv;
  uint8_t* ctx_codes = tp.ctx_codes ? tp.ctx_codes : ws.ctx_codes;
  float* ctx_scales = tp.ctx_scales ? tp.ctx_scales : ws.ctx_scales;
  uint16_t* h1 = tp.h1 ? tp.h1 : ws.h1;
  uint8_t* h1_codes = tp.h1_codes ? tp.h1_codes : ws.h1_codes;
  float* h1_scales = tp.h1_scales ? tp.h1_scales : ws.h1_scales;
  uint8_t* f_codes = tp.f_codes ? tp.f_codes : ws.f_codes;
  float* f_scales = tp.f_scales ? tp.f_scales : ws.f_scales;
  float* ctx_zeros = tp.ctx_zeros ? tp.ctx_zeros : ws.ctx_zeros;
  float* h1_zeros = tp.h1_zeros ? tp.h1_zeros : ws.h1_zeros;
  float* f_zeros = tp.f_zeros ? tp.f_zeros : ws.f_zeros;

  // asymmetric layer: (codes, scales, zeros) -> linear with the weight code sums; the
  // requantizing epilogues write asymmetric codes (e.out_zeros set by the caller)
  auto alin = [&](const uint8_t* ac, const float* as, const float* az, const uint8_t* wc, const float* wsc,
                  const float* wsum, int64_t N, int64_t K, q4_epilogue e) -> q4_status {
    return q4_w4a4_asym_linear(ac, as, az, wc, wsc, wsum, M, N, K, &e, ws.gemm_ws, ws.gemm_ws_bytes, stream);
  };
  auto aacc_tap = [&](const uint8_t* ac, const float* as, const float* az, const uint8_t* wc, const float* wsc,
                      int64_t N, int64_t K, int32_t* out, const int8_t* w8) -> q4_status {
    if (!out) return Q4_OK;
    q4_epilogue e;
    memset(&e, 0, sizeof e);
    e.kind = Q4_EPI_I32;
    e.out_i32 = out;
    e.w_i8 = w8;
    return q4_w4a4_asym_linear(ac, as, az, wc, wsc, nullptr, M, N, K, &e, nullptr, 0, stream);
  };
  auto lin = [&](const uint8_t* ac, const float* as, const uint8_t* wc, const float* wsc, int64_t N, int64_t K,
                 q4_epilogue e) -> q4_status {
    if (i8) {
      e.w_i8 = nullptr;
      return q4_w8a8_linear(reinterpret_cast<const int8_t*>(ac), as, reinterpret_cast<const int8_t*>(wc), wsc, M, N, K,
                            &e, ws.gemm_ws, ws.gemm_ws_bytes, stream);
    }
    return q4_w4a4_linear(ac, as, wc, wsc, M, N, K, &e, ws.gemm_ws, ws.gemm_ws_bytes, stream);
  };
  // INT32 tap of a part: the same operands through the mainloop its production launch runs
  // (prepacked weights when present; the 1-CTA mainloop for the row-epilogue parts, which the
  // pair mainloop does not take), so the tap sees the accumulators the epilogue consumed.
  auto acc_tap = [&](const uint8_t* ac, const float* as, const uint8_t* wc, const float* wsc, int64_t N, int64_t K,
                     int32_t* out, const int8_t* w8, bool row_epi) -> q4_status {
    if (!out) return Q4_OK;
    q4_epilogue e;
    memset(&e, 0, sizeof e);
    e.kind = Q4_EPI_I32;
    e.out_i32 = out;
    if (w8) {
      e.w_i8 = w8;
      e.mainloop = row_epi ? Q4_MAINLOOP_TCGEN05_W8_1CTA : Q4_MAINLOOP_TCGEN05_W8;
    }
    if (i8)
      return q4_w8a8_linear(reinterpret_cast<const int8_t*>(ac), as, reinterpret_cast<const int8_t*>(wc), wsc, M, N, K,
                            &e, nullptr, 0, stream);
    return q4_w4a4_linear(ac, as, wc, wsc, M, N, K, &e, nullptr, 0, stream);
  };
  // an FP16 part (strategy bit set): fp16 activation x fp16 weight, same epilogue
  auto f16lin = [&](const uint16_t* a, const uint16_t* wf, int64_t N, int64_t K, q4_epilogue e) -> q4_status {
    e.w_i8 = nullptr;
    return q4_f16_linear(a, wf, M, N, K, &e, ws.gemm_ws, ws.gemm_ws_bytes, stream);
  };
  uint16_t* ctx_f16 = tp.ctx ? tp.ctx : ws.ctx;
  uint16_t* ffn1 = tp.ffn1 ? tp.ffn1 : ws.ffn1;  // NULL unless tapped or the MLP output is FP16
  q4_epilogue e;
  // QKV projection: dequant + bias -> fp16
  memset(&e, 0, sizeof e);
  e.kind = Q4_EPI_F16; e.bias = w->bqkv; e.out_f16 = qkv; e.w_i8 = w->wqkv8;
  if (asym) {
    if ((st = alin(hq_in, hs_in, hz_in, w->wqkv, w->sqkv, w->cqkv, 3 * h, h, e))) return st;
    if ((st = aacc_tap(hq_in, hs_in, hz_in, w->wqkv, w->sqkv, 3 * h, h, tp.acc_qkv, w->wqkv8))) return st;
  } else if (fp & 1) {
    if ((st = f16lin(h_in, w->fqkv, 3 * h, h, e))) return st;
  } else {
    if ((st = lin(hq_in, hs_in, w->wqkv, w->sqkv, 3 * h, h, e))) return st;
    if ((st = acc_tap(hq_in, hs_in, w->wqkv, w->sqkv, 3 * h, h, tp.acc_qkv, w->wqkv8, false))) return st;
  }
  // FP16 attention + fused per-token ctx quantize
  if ((st = i8     ? q4_attention_f16_q8(qkv, B, S, cfg->heads, cfg->head_dim, ctx_f16,
                                         reinterpret_cast<int8_t*>(ctx_codes), ctx_scales, stream)
            : asym ? q4_attention_f16_q4_asym(qkv, B, S, cfg->heads, cfg->head_dim, ctx_f16, ctx_codes, ctx_scales,
                                              ctx_zeros, stream)
                   : q4_attention_f16_q4(qkv, B, S, cfg->heads, cfg->head_dim, ctx_f16, ctx_codes, ctx_scales, stream)))
    return st;
  // attention output: dequant + bias + residual(h_in) + LN1 + requant
  memset(&e, 0, sizeof e);
  e.kind = Q4_EPI_RESLN_Q4; e.bias = w->bo; e.residual = h_in; e.gamma = w->ln1_g; e.beta = w->ln1_b;
  e.ln_eps = cfg->ln_eps; e.out_f16 = h1; e.out_codes = h1_codes; e.out_scales = h1_scales; e.w_i8 = w->wo8;
  if (asym) {
    e.out_zeros = h1_zeros;
    if ((st = alin(ctx_codes, ctx_scales, ctx_zeros, w->wo, w->so, w->co, h, h, e))) return st;
    if ((st = aacc_tap(ctx_codes, ctx_scales, ctx_zeros, w->wo, w->so, h, h, tp.acc_o, w->wo8))) return st;
  } else if (fp & 2) {
    if ((st = f16lin(ctx_f16, w->fo, h, h, e))) return st;
  } else {
    if ((st = lin(ctx_codes, ctx_scales, w->wo, w->so, h, h, e))) return st;
    if ((st = acc_tap(ctx_codes, ctx_scales, w->wo, w->so, h, h, tp.acc_o, w->wo8, true))) return st;
  }
  // MLP intermediate: dequant + bias + GELU + requant (+ fp16 output for an FP16 MLP output)
  memset(&e, 0, sizeof e);
  e.kind = Q4_EPI_GELU_Q4; e.bias = w->b1; e.out_f16 = ffn1; e.out_codes = f_codes; e.out_scales = f_scales;
  e.w_i8 = w->w18;
  if (asym) {
    e.out_zeros = f_zeros;
    if ((st = alin(h1_codes, h1_scales, h1_zeros, w->w1, w->s1, w->c1, f, h, e))) return st;
    if ((st = aacc_tap(h1_codes, h1_scales, h1_zeros, w->w1, w->s1, f, h, tp.acc_1, w->w18))) return st;
  } else if (fp & 4) {
    if ((st = f16lin(h1, w->f1, f, h, e))) return st;
  } else {
    if ((st = lin(h1_codes, h1_scales, w->w1, w->s1, f, h, e))) return st;
    if ((st = acc_tap(h1_codes, h1_scales, w->w1, w->s1, f, h, tp.acc_1, w->w18, true))) return st;
  }
  // MLP output: dequant + bias + residual(h1) + LN2 + requant
  memset(&e, 0, sizeof e);
  e.kind = Q4_EPI_RESLN_Q4; e.bias = w->b2; e.residual = h1; e.gamma = w->ln2_g; e.beta = w->ln2_b;
  e.ln_eps = cfg->ln_eps; e.out_f16 = h_out; e.out_codes = hq_out; e.out_scales = hs_out; e.w_i8 = w->w28;
  if (asym) {
    e.out_zeros = hz_out;
    if ((st = alin(f_codes, f_scales, f_zeros, w->w2, w->s2, w->c2, h, f, e))) return st;
    if ((st = aacc_tap(f_codes, f_scales, f_zeros, w->w2, w->s2, h, f, tp.acc_2, w->w28))) return st;
  } else if (fp & 8) {
    if ((st = f16lin(ffn1, w->f2, h, f, e))) return st;
  } else {
    if ((st = lin(f_codes, f_scales, w->w2, w->s2, h, f, e))) return st;
    if ((st = acc_tap(f_codes, f_scales, w->w2, w->s2, h, f, tp.acc_2, w->w28, true))) return st;
  }
  return Q4_OK;
}
}  // namespace

extern "C" {

q4_status q4_encoder_layer(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B, int64_t S,
                           const uint16_t* h_in, const uint8_t* hq_in, const float* hs_in, uint16_t* h_out,
                           uint8_t* hq_out, float* hs_out, void* workspace, size_t ws_bytes, const q4_taps* taps,
                           void* stream) {
  g_err[0] = 0;
  if (cfg && cfg->asym_acts) return fail(Q4_EINVAL, "q4_encoder_layer: asym_acts set (use q4_encoder_layer_asym)");
  return encoder_layer_impl(cfg, w, B, S, h_in, hq_in, hs_in, h_out, hq_out, hs_out, workspace, ws_bytes, taps,
                            stream, false);
}

q4_status q4_encoder_layer_asym(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B, int64_t S,
                                const uint16_t* h_in, const uint8_t* hq_in, const float* hs_in, const float* hz_in,
                                uint16_t* h_out, uint8_t* hq_out, float* hs_out, float* hz_out, void* workspace,
                                size_t ws_bytes, const q4_taps* taps, void* stream) {
  g_err[0] = 0;
  if (!cfg || !cfg->asym_acts) return fail(Q4_EINVAL, "q4_encoder_layer_asym: cfg->asym_acts must be 1");
  return encoder_layer_impl(cfg, w, B, S, h_in, hq_in, hs_in, h_out, hq_out, hs_out, workspace, ws_bytes, taps, stream,
                            false, hz_in, hz_out);
}

q4_status q4_encoder_layer_w8a8(const q4_layer_cfg* cfg, const q4_layer_weights* w, int64_t B, int64_t S,
                                const uint16_t* h_in, const int8_t* hq_in, const float* hs_in, uint16_t* h_out,
                                int8_t* hq_out, float* hs_out, void* workspace, size_t ws_bytes, const q4_taps* taps,
                                void* stream) {
  g_err[0] = 0;
  return encoder_layer_impl(cfg, w, B, S, h_in, reinterpret_cast<const uint8_t*>(hq_in), hs_in, h_out,
                            reinterpret_cast<uint8_t*>(hq_out), hs_out, workspace, ws_bytes, taps, stream, true);
}

// ------------------------------------------------------------------ encoder stack

namespace {
struct StackWs {
  uint16_t* hid[2];
  uint8_t* hq[2];
  float* hs[2];
  float* hz[2];  // asymmetric activations: zero points
  uint8_t* layer;
  size_t layer_bytes, bytes;
};
StackWs stack_ws(const q4_layer_cfg* c, int64_t M, uint8_t* base, bool i8 = false) {
  StackWs w;
  size_t o = 0;
  auto take = [&](size_t n) { size_t r = o; o = align_up(o + n); return base ? base + r : nullptr; };
  for (int i = 0; i < 2; ++i) {
    w.hid[i] = (uint16_t*)take((size_t)M * c->hidden * 2);
    w.hq[i] = take((size_t)M * c->hidden / (i8 ? 1 : 2));
    w.hs[i] = (float*)take((size_t)M * 4);
    w.hz[i] = (!i8 && c->asym_acts) ? (float*)take((size_t)M * 4) : nullptr;
  }
  w.layer_bytes = layer_ws(c, M, nullptr, i8).bytes;
  w.layer = take(w.layer_bytes);
  w.bytes = o;
  return w;
}
bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

q4_status encoder_stack_impl(const q4_layer_cfg* cfg, const q4_layer_weights* layers, int32_t L, int64_t B,
                             int64_t S, const uint16_t* h_in, uint16_t* h_out, void* workspace, size_t ws_bytes,
                             void* stream, bool i8) {
  const char* who = i8 ? "q4_encoder_stack_w8a8" : "q4_encoder_stack";
  q4_status st = check_cfg(cfg, who);
  if (st) return st;
  if (L < 1 || !layers) return fail(Q4_EINVAL, "%s: L=%d layers=%p", who, L, (const void*)layers);
  if (B < 0 || S < 1 || S > 128) return fail(Q4_ESHAPE, "%s: B=%lld S=%lld", who, (long long)B, (long long)S);
  const int64_t M = B * S, h = cfg->hidden;
  if (M == 0) return Q4_OK;
  if (!h_in || !h_out) return fail(Q4_EINVAL, "%s: NULL h_in/h_out", who);
  StackWs ws = stack_ws(cfg, M, (uint8_t*)workspace, i8);
  if (!workspace || ws_bytes < ws.bytes)
    return fail(Q4_EINVAL, "%s: workspace %zu bytes < required %zu", who, ws_bytes, ws.bytes);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t hbytes = (size_t)M * h * 2;
  const uint16_t* x = h_in;
  if (!is_device_ptr(h_in)) {  // end-to-end entry: host input copied inside the call
    cudaError_t e = cudaMemcpyAsync(ws.hid[1], h_in, hbytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "q4_encoder_stack: H2D copy");
    x = ws.hid[1];
  } else if (!al16(h_in)) {
    return fail(Q4_EALIGN, "q4_encoder_stack: h_in must be 16-byte aligned");
  }
  // layer-0 activation quantize (the only standalone quantize in the forward)
  if (i8 && cfg->asym_acts) return fail(Q4_EUNSUPPORTED, "%s: asym_acts on the W8A8 baseline", who);
  if ((st = i8               ? q4_quantize_rows_i8(x, M, h, h, 0.f, reinterpret_cast<int8_t*>(ws.hq[1]), ws.hs[1], stream)
            : cfg->asym_acts ? q4_quantize_rows_asym(x, M, h, h, ws.hq[1], ws.hs[1], ws.hz[1], stream)
                             : q4_quantize_rows(x, M, h, h, 0.f, ws.hq[1], ws.hs[1], stream)))
    return st;
  const bool out_dev = is_device_ptr(h_out);
  for (int l = 0; l < L; ++l) {
    const int o = l & 1;
    const uint16_t* hin = (l == 0) ? x : ws.hid[1 - o];
    uint16_t* hout = (l == L - 1 && out_dev) ? h_out : ws.hid[o];
    if ((st = encoder_layer_impl(cfg, &layers[l], B, S, hin, ws.hq[1 - o], ws.hs[1 - o], hout, ws.hq[o], ws.hs[o],
                                 ws.layer, ws.layer_bytes, nullptr, stream, i8, ws.hz[1 - o], ws.hz[o])))
      return st;
  }
  if (!out_dev) {
    cudaError_t e = cudaMemcpyAsync(h_out, ws.hid[(L - 1) & 1], hbytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "q4_encoder_stack: D2H copy");
  }
  return Q4_OK;
}
}  // namespace

size_t q4_encoder_stack_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S) {
  if (!cfg) return 0;
  return stack_ws(cfg, B * S, nullptr).bytes;
}
size_t q4_encoder_stack_w8a8_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S) {
  if (!cfg) return 0;
  return stack_ws(cfg, B * S, nullptr, true).bytes;
}

q4_status q4_encoder_stack(const q4_layer_cfg* cfg, const q4_layer_weights* layers, int32_t L, int64_t B, int64_t S,
                           const uint16_t* h_in, uint16_t* h_out, void* workspace, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  return encoder_stack_impl(cfg, layers, L, B, S, h_in, h_out, workspace, ws_bytes, stream, false);
}
q4_status q4_encoder_stack_w8a8(const q4_layer_cfg* cfg, const q4_layer_weights* layers, int32_t L, int64_t B,
                                int64_t S, const uint16_t* h_in, uint16_t* h_out, void* workspace, size_t ws_bytes,
                                void* stream) {
  g_err[0] = 0;
  return encoder_stack_impl(cfg, layers, L, B, S, h_in, h_out, workspace, ws_bytes, stream, true);
}

// ------------------------------------------------------------------ pipelined host-buffer serving
// nbatch batches of host (pinned) inputs -> host outputs.  Batch i's H2D copy runs on a copy-in
// stream, its forward on the caller's stream, its D2H copy on a copy-out stream; two device
// input and two device output buffers (slot = i % 2) let batch i+1's upload and batch i-1's
// download overlap batch i's forward.  The copy streams and events are created per call (the
// call allocates no device memory) so concurrent calls on one device share no state.
size_t q4_encoder_pipeline_workspace(const q4_layer_cfg* cfg, int64_t B, int64_t S) {
  if (!cfg) return 0;
  const size_t hb = align_up((size_t)(B * S) * cfg->hidden * 2);
  return stack_ws(cfg, B * S, nullptr).bytes + 4 * hb;
}

q4_status q4_encoder_pipeline(const q4_layer_cfg* cfg, const q4_layer_weights* layers, int32_t L, int64_t B, int64_t S,
                              const uint16_t* const* h_in, uint16_t* const* h_out, int32_t nbatch, void* workspace,
                              size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  q4_status st = check_cfg(cfg, "q4_encoder_pipeline");
  if (st) return st;
  if (nbatch < 0 || (nbatch > 0 && (!h_in || !h_out))) return fail(Q4_EINVAL, "q4_encoder_pipeline: nbatch=%d h_in/h_out", nbatch);
  const size_t need = q4_encoder_pipeline_workspace(cfg, B, S);
  if (!workspace || ws_bytes < need)
    return fail(Q4_EINVAL, "q4_encoder_pipeline: workspace %zu bytes < required %zu", ws_bytes, need);
  if (nbatch == 0 || B * S == 0) return Q4_OK;
  const size_t stack_bytes = stack_ws(cfg, B * S, nullptr).bytes;
  const size_t hbytes = (size_t)(B * S) * cfg->hidden * 2, hb = align_up(hbytes);
  uint8_t* base = (uint8_t*)workspace;
  uint16_t* din[2] = {(uint16_t*)(base + stack_bytes), (uint16_t*)(base + stack_bytes + hb)};
  uint16_t* dout[2] = {(uint16_t*)(base + stack_bytes + 2 * hb), (uint16_t*)(base + stack_bytes + 3 * hb)};
  // Streams and events belong to this call (re-entrant: concurrent calls share nothing).  They
  // are destroyed before returning; CUDA releases them once the enqueued work that uses them
  // has completed (cudaStreamDestroy / cudaEventDestroy on pending work return immediately).
  struct Aux {
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t ev[9] = {};  // in_ready[2], in_free[2], done[2], out_free[2], start
    ~Aux() {
      for (cudaEvent_t x : ev)
        if (x) cudaEventDestroy(x);
      if (cin) cudaStreamDestroy(cin);
      if (cout) cudaStreamDestroy(cout);
    }
  } a;
  {
    cudaError_t e = cudaStreamCreateWithFlags(&a.cin, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a.cout, cudaStreamNonBlocking);
    for (int k = 0; k < 9 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&a.ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "q4_encoder_pipeline: stream/event creation");
  }
  cudaEvent_t* in_ready = a.ev;
  cudaEvent_t* in_free = a.ev + 2;
  cudaEvent_t* done = a.ev + 4;
  cudaEvent_t* out_free = a.ev + 6;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  // the auxiliary streams start after everything already queued on the caller's stream
  cudaEvent_t start = a.ev[8];
  if ((e = cudaEventRecord(start, s)) != cudaSuccess) return cuda_fail(e, "q4_encoder_pipeline");
  cudaStreamWaitEvent(a.cin, start, 0);
  cudaStreamWaitEvent(a.cout, start, 0);
  for (int32_t i = 0; i < nbatch; ++i) {
    const int k = i & 1;
    if (i >= 2) cudaStreamWaitEvent(a.cin, in_free[k], 0);  // batch i-2 has consumed din[k]
    if ((e = cudaMemcpyAsync(din[k], h_in[i], hbytes, cudaMemcpyHostToDevice, a.cin)) != cudaSuccess)
      return cuda_fail(e, "q4_encoder_pipeline: H2D");
    cudaEventRecord(in_ready[k], a.cin);
    cudaStreamWaitEvent(s, in_ready[k], 0);
    if (i >= 2) cudaStreamWaitEvent(s, out_free[k], 0);  // batch i-2's download has read dout[k]
    if ((st = encoder_stack_impl(cfg, layers, L, B, S, din[k], dout[k], workspace, stack_bytes, stream, false)))
      return st;
    cudaEventRecord(in_free[k], s);
    cudaEventRecord(done[k], s);
    cudaStreamWaitEvent(a.cout, done[k], 0);
    if ((e = cudaMemcpyAsync(h_out[i], dout[k], hbytes, cudaMemcpyDeviceToHost, a.cout)) != cudaSuccess)
      return cuda_fail(e, "q4_encoder_pipeline: D2H");
    cudaEventRecord(out_free[k], a.cout);
  }
  // the caller's stream completes after the last download
  cudaStreamWaitEvent(s, out_free[(nbatch - 1) & 1], 0);
  e = cudaGetLastError();
  return e == cudaSuccess ? Q4_OK : cuda_fail(e, "q4_encoder_pipeline");
}

}  // extern "C"

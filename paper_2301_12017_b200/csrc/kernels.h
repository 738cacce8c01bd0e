// kernels.h -- internal launch helpers of the CUDA path (not part of the C ABI).
#pragma once
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace q4 {

void note_launch(int n = 1);  // counts kernels launched (q4_launch_count)

// Profiling knobs (Q4_DEBUG_SKIP, Q4_TRACE, Q4_TN, Q4_PAIR, Q4_NO_PDL, Q4_ATTN_DBG) exist only in
// a build compiled with -DQ4_PROFILING (build.py --profiling -> libq4_prof.so, selected with
// Q4_LIB_PATH).  The shipped libq4.so reads no environment variable: prof_env() is nullptr.
#ifdef Q4_PROFILING
inline const char* prof_env(const char* name) { return getenv(name); }
#else
inline const char* prof_env(const char*) { return nullptr; }
#endif

// Launch with programmatic stream serialization (PDL) when `pdl`: the kernel may start
// while its predecessor in the stream drains (it calls pdl_wait() before dependent
// accesses; without the attribute that wait is a no-op).  Callers enable it for small
// problems only (kPdlMaxRows): at batch 1-8 it cuts BERT-base latency 5-13%, at the
// BERT-large batch-256 step it costs 4% (measured; early-resident dependents of the
// long persistent kernels), see DESIGN.md.
constexpr int64_t kPdlMaxRows = 8192;
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const bool off = prof_env("Q4_NO_PDL") != nullptr;  // profiling only: plain launches
  cfg.numAttrs = (pdl && !off) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

struct GemmArgs {
  const uint8_t* a_codes;  // [M, K/2]
  const int8_t* a_i8;      // W8A8: int8 activation codes [M, K] (then w_i8 holds int8 weight codes
                           // in natural K order and requant kinds write int8 codes [M, N]); else nullptr
  const float* a_zeros = nullptr;  // asymmetric activations: per-row zero point; a_codes unsigned nibbles
  const float* w_sums = nullptr;   // with a_zeros: per-output-channel weight-code sums (as float)
  float* out_zeros = nullptr;      // GELU_Q4 / RESLN_Q4: asymmetric requant output (zero points)
  bool f16_ops = false;    // with a_i8 / w_i8 pointing at fp16 [M, K] / [N, K] and K counted in
                           // bytes (2 x elements): kind::f16 MMA, unit scales, INT4 requant
  const float* a_scales;   // [M]
  const uint8_t* w_codes;  // [N, K/2]
  const int8_t* w_i8;      // [N, K] prepacked int8 (q4_prepack_weights) or nullptr
  const float* w_scales;   // [N]
  int M, N, K;
  int kind;      // q4_epi_kind
  int mainloop;  // q4_mainloop
  const __half* bias;
  const __half* residual;
  const __half* gamma;
  const __half* beta;
  float ln_eps, clip;
  int32_t* out_i32;
  __half* out_f16;
  uint8_t* out_codes;
  float* out_scales;
};

cudaError_t launch_prepack_weights(const uint8_t* w_codes, int64_t N, int64_t K, int8_t* w_i8, cudaStream_t s);
cudaError_t launch_quantize_rows_asym(const __half* x, int64_t rows, int cols, int64_t ld_x, uint8_t* codes,
                                      float* scales, float* zeros, cudaStream_t s);
cudaError_t launch_weight_code_sums(const uint8_t* w_codes, int64_t N, int64_t K, float* sums, cudaStream_t s);
cudaError_t launch_quantize_rows(const __half* x, int64_t rows, int cols, int64_t ld_x, float clip,
                                 uint8_t* codes, float* scales, cudaStream_t s);
cudaError_t launch_quantize_rows_i8(const __half* x, int64_t rows, int cols, int64_t ld_x, float clip,
                                    int8_t* codes, float* scales, cudaStream_t s);
// Returns cudaErrorNotSupported for shapes the tcgen05 path cannot take (message in *why).
// Row epilogues (GELU_Q4 / RESLN_Q4) need `ws` of tc_workspace_bytes(M, N, tc_tile_n(...)).
cudaError_t launch_w4a4_tc(const GemmArgs& g, void* ws, size_t ws_bytes, cudaStream_t s, const char** why);
int tc_tile_n(int M, int N, int kind);
size_t tc_workspace_bytes(int M, int N, int TN, int kind);
size_t tc_row_grid(int M, int N, int TN);  // CTAs of a 1-CTA row-epilogue launch
size_t tc_counter_bytes(int M);  // the rendezvous counters at the start of a row-epilogue workspace
cudaError_t launch_floor_kernel(int ctas, cudaStream_t s);  // (declared below the GEMM args too)
// NEXT-4: 2:4-sparse W4A4 (gemm_sparse.cu)
struct SparseArgs {
  const uint8_t* a_codes;  // [M, K/2] packed INT4 activations
  const float* a_scales;   // [M]
  const int8_t* w_vals;    // [N, K/2] compressed 16*q weights (two kept values per group of four)
  const uint32_t* w_meta;  // [N, K/32] 2:4 position nibbles
  const float* w_scales;   // [N]
  const __half* bias;      // [N] or nullptr
  int M, N, K;
  int32_t* out_i32;        // I32 epilogue (exclusive with out_f16)
  __half* out_f16;         // F16 epilogue
};
cudaError_t launch_w4a4_sparse24(const SparseArgs& a, cudaStream_t s, const char** why);
cudaError_t launch_prune24(const __half* w, int64_t N, int64_t K, __half* out, cudaStream_t s);
cudaError_t launch_sparse24_compress(const uint8_t* codes, int64_t N, int64_t K, int8_t* vals, uint32_t* meta,
                                     int* violations, cudaStream_t s);  // empty PDL kernel (measurement only)
cudaError_t launch_w4a4_legacy(const GemmArgs& g, bool s4, cudaStream_t s, const char** why);
// i8: W8A8 baseline -- int8 ctx codes [B*S, h] with scale amax/127 instead of packed INT4
cudaError_t launch_attention_tc(const __half* qkv, int B, int S, int heads, __half* ctx_f16,
                                uint8_t* ctx_codes, float* ctx_scales, cudaStream_t s, bool i8 = false,
                                float* ctx_zeros = nullptr);

}  // namespace q4

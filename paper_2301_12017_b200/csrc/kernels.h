// kernels.h -- internal launch helpers of the CUDA path (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace q4 {

void note_launch(int n = 1);  // counts kernels launched (q4_launch_count)

struct GemmArgs {
  const uint8_t* a_codes;  // [M, K/2]
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
cudaError_t launch_quantize_rows(const __half* x, int64_t rows, int cols, int64_t ld_x, float clip,
                                 uint8_t* codes, float* scales, cudaStream_t s);
// Returns cudaErrorNotSupported for shapes the tcgen05 path cannot take (message in *why).
// Row epilogues (GELU_Q4 / RESLN_Q4) need `ws` of tc_workspace_bytes(M, N, tc_tile_n(...)).
cudaError_t launch_w4a4_tc(const GemmArgs& g, void* ws, size_t ws_bytes, cudaStream_t s, const char** why);
int tc_tile_n(int M, int N, int kind);
size_t tc_workspace_bytes(int M, int N, int TN);
cudaError_t launch_w4a4_legacy(const GemmArgs& g, bool s4, cudaStream_t s, const char** why);
cudaError_t launch_attention(const __half* qkv, int B, int S, int heads, __half* ctx_f16,
                             uint8_t* ctx_codes, float* ctx_scales, cudaStream_t s);
cudaError_t launch_attention_tc(const __half* qkv, int B, int S, int heads, __half* ctx_f16,
                                uint8_t* ctx_codes, float* ctx_scales, cudaStream_t s);

}  // namespace q4

// quantize.cu -- a1/a2: symmetric per-row INT4 quantize + pack (PAPER.md:703-708,
// 517-522; readings R1-R3, R5, R10).  Memory-bound: 2 B/elem in, 0.5 B/elem + 4 B/row out.
// Also the 8-bit variant of the W8A8 baseline (int8 codes, 1 B/elem out; oracle O-11).
//
// One warp per row.  Each lane owns 16-byte vectors (8 halves) v = lane + 32*i, kept
// in registers between the two passes (warp-shuffle max-abs, then codes), so x is read
// from HBM exactly once.  Codes: round-half-even of the rational 7x/amax (R3),
// computed as rint(x * RN(7/amax)) with an exact FMA tie-break near half-integers
// (requant8 in common.cuh) -- bit-identical to rint(div.rn(7x, amax)).
#include "kernels.h"

namespace q4 {

// I8: the W8A8 variant (oracle O-11): int8 codes, one per byte, scale amax/127.
template <int MAXV, bool I8>
__global__ void __launch_bounds__(256) quantize_rows_kernel(const __half* __restrict__ x,
                                                            int64_t rows, int cols, int64_t ld_x,
                                                            float clip, uint8_t* __restrict__ codes,
                                                            float* __restrict__ scales) {
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nvec = cols >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * ld_x);
  uint4 v[MAXV];
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int vi = lane + 32 * i;
    if (vi < nvec) {
      v[i] = __ldg(xr + vi);
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = unpack_half2(u[j]);
        if (clip > 0.f) {
          f.x = fminf(fmaxf(f.x, -clip), clip);
          f.y = fminf(fmaxf(f.y, -clip), clip);
        }
        amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  constexpr float QM = I8 ? 127.0f : 7.0f;
  const float rq = amax > 0.f ? __fdiv_rn(QM, amax) : 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int vi = lane + 32 * i;
    if (vi < nvec) {
      const uint32_t hh[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
      if constexpr (I8)
        reinterpret_cast<uint2*>(codes + row * (int64_t)cols)[vi] = requant8_i8(hh, amax, rq, clip);
      else
        reinterpret_cast<uint32_t*>(codes + row * (int64_t)(cols >> 1))[vi] = requant8(hh, amax, rq, clip);
    }
  }
  if (lane == 0) scales[row] = amax > 0.f ? __fdiv_rn(amax, QM) : 1.0f;
}

// Rows longer than 32*16*8 = 4096: two passes over global memory.
template <bool I8>
__global__ void __launch_bounds__(256) quantize_rows_long_kernel(const __half* __restrict__ x,
                                                                 int64_t rows, int cols,
                                                                 int64_t ld_x, float clip,
                                                                 uint8_t* __restrict__ codes,
                                                                 float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nvec = cols >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * ld_x);
  float amax = 0.f;
  for (int vi = lane; vi < nvec; vi += 32) {
    uint4 vv = __ldg(xr + vi);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&vv);
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_half2(u[j]);
      if (clip > 0.f) {
        f.x = fminf(fmaxf(f.x, -clip), clip);
        f.y = fminf(fmaxf(f.y, -clip), clip);
      }
      amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  constexpr float QM = I8 ? 127.0f : 7.0f;
  const float rq = amax > 0.f ? __fdiv_rn(QM, amax) : 0.f;
  for (int vi = lane; vi < nvec; vi += 32) {
    const uint4 vv = __ldg(xr + vi);
    const uint32_t hh[4] = {vv.x, vv.y, vv.z, vv.w};
    if constexpr (I8)
      reinterpret_cast<uint2*>(codes + row * (int64_t)cols)[vi] = requant8_i8(hh, amax, rq, clip);
    else
      reinterpret_cast<uint32_t*>(codes + row * (int64_t)(cols >> 1))[vi] = requant8(hh, amax, rq, clip);
  }
  if (lane == 0) scales[row] = amax > 0.f ? __fdiv_rn(amax, QM) : 1.0f;
}

// Offline weight prep for the tcgen05 mainloop: packed INT4 [N, K/2] -> int8 [N, K] holding
// 16*q in the operand K order the on-chip activation unpack produces: each 16-byte packed
// chunk (32 consecutive k) -> 16 bytes of the even k, then 16 bytes of the odd k (the
// K-permutation trick).  Same codes, same products.
__global__ void prepack_weights_kernel(const uint4* __restrict__ w, int64_t nchunks, uint4* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nchunks) return;
  const uint4 x = __ldg(w + i);
  out[2 * i] = make_uint4(nib_lo16(x.x), nib_lo16(x.y), nib_lo16(x.z), nib_lo16(x.w));
  out[2 * i + 1] = make_uint4(nib_hi16(x.x), nib_hi16(x.y), nib_hi16(x.z), nib_hi16(x.w));
}

cudaError_t launch_prepack_weights(const uint8_t* w_codes, int64_t N, int64_t K, int8_t* w_i8, cudaStream_t s) {
  const int64_t nchunks = N * K / 32;
  if (nchunks == 0) return cudaSuccess;
  note_launch();
  prepack_weights_kernel<<<(unsigned)((nchunks + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(w_codes), nchunks, reinterpret_cast<uint4*>(w_i8));
  return cudaGetLastError();
}

// Asymmetric per-token INT4 (NEXT-3, oracle O-15, readings R17/R18):
// zero = min, q = rhe(15 (x - min) / (max - min)) in [0, 15], scale = fl32(fl64(max-min)/15).
// x - min and max - min of two fp16 values are exact in fp64 (<= 41 significant bits), so
// p = d * (15/D) in fp64 is within 1e-14 of the rational; near a half-integer the exact
// fp64 residual 15 d - D h (both products exact) decides.  Warp per row, one HBM read.
template <int MAXV>
__global__ void __launch_bounds__(256) quantize_rows_asym_kernel(const __half* __restrict__ x, int64_t rows, int cols,
                                                                 int64_t ld_x, uint8_t* __restrict__ codes,
                                                                 float* __restrict__ scales, float* __restrict__ zeros) {
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nvec = cols >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * ld_x);
  uint4 v[MAXV];
  float mn = INFINITY, mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int vi = lane + 32 * i;
    if (vi < nvec) {
      v[i] = __ldg(xr + vi);
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_half2(u[j]);
        mn = fminf(mn, fminf(f.x, f.y));
        mx = fmaxf(mx, fmaxf(f.x, f.y));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const double D = (double)mx - (double)mn;
  const double r15 = D > 0.0 ? 15.0 / D : 0.0;
  uint32_t* cr = reinterpret_cast<uint32_t*>(codes + row * (int64_t)(cols >> 1));
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int vi = lane + 32 * i;
    if (vi < nvec) {
      uint32_t w = 0;
      if (D > 0.0) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_half2(u[j]);
          w |= asym_code(f.x, (double)mn, D, r15) << (8 * j);
          w |= asym_code(f.y, (double)mn, D, r15) << (8 * j + 4);
        }
      }
      cr[vi] = w;
    }
  }
  if (lane == 0) {
    scales[row] = D > 0.0 ? (float)(D / 15.0) : 1.0f;
    zeros[row] = mn;
  }
}

// Per-output-channel sum of the INT4 weight codes (asymmetric activations' zero-point term).
__global__ void weight_code_sums_kernel(const uint8_t* __restrict__ w, int64_t N, int64_t kb, float* __restrict__ sums) {
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  int s = 0;
  for (int64_t j = lane; j < kb; j += 32) {
    const uint32_t b = w[n * kb + j];
    s += ((int)(b << 28) >> 28) + ((int)(b << 24) >> 28);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sums[n] = (float)s;
}

cudaError_t launch_quantize_rows_asym(const __half* x, int64_t rows, int cols, int64_t ld_x, uint8_t* codes,
                                      float* scales, float* zeros, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const int warps = 8;
  const dim3 grid((unsigned)((rows + warps - 1) / warps)), block(32 * warps);
  const int nvec = cols / 8;
  const bool pdl = rows <= kPdlMaxRows;
  note_launch();
  if (nvec <= 32) return launch_pdl(pdl, quantize_rows_asym_kernel<1>, grid, block, 0, s, x, rows, cols, ld_x, codes, scales, zeros);
  if (nvec <= 64) return launch_pdl(pdl, quantize_rows_asym_kernel<2>, grid, block, 0, s, x, rows, cols, ld_x, codes, scales, zeros);
  if (nvec <= 128) return launch_pdl(pdl, quantize_rows_asym_kernel<4>, grid, block, 0, s, x, rows, cols, ld_x, codes, scales, zeros);
  if (nvec <= 512) return launch_pdl(pdl, quantize_rows_asym_kernel<16>, grid, block, 0, s, x, rows, cols, ld_x, codes, scales, zeros);
  return cudaErrorNotSupported;
}

cudaError_t launch_weight_code_sums(const uint8_t* w_codes, int64_t N, int64_t K, float* sums, cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  note_launch();
  weight_code_sums_kernel<<<(unsigned)((N + 7) / 8), 256, 0, s>>>(w_codes, N, K / 2, sums);
  return cudaGetLastError();
}

template <bool I8>
static cudaError_t launch_quantize_impl(const __half* x, int64_t rows, int cols, int64_t ld_x, float clip,
                                        uint8_t* codes, float* scales, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const int warps = 8;
  const dim3 grid((unsigned)((rows + warps - 1) / warps)), block(32 * warps);
  const int nvec = cols / 8;
  const bool pdl = rows <= kPdlMaxRows;
  note_launch();
  if (nvec <= 32) return launch_pdl(pdl, quantize_rows_kernel<1, I8>, grid, block, 0, s, x, rows, cols, ld_x, clip, codes, scales);
  else if (nvec <= 64) return launch_pdl(pdl, quantize_rows_kernel<2, I8>, grid, block, 0, s, x, rows, cols, ld_x, clip, codes, scales);
  else if (nvec <= 128) return launch_pdl(pdl, quantize_rows_kernel<4, I8>, grid, block, 0, s, x, rows, cols, ld_x, clip, codes, scales);
  else if (nvec <= 256) quantize_rows_kernel<8, I8><<<grid, block, 0, s>>>(x, rows, cols, ld_x, clip, codes, scales);
  else if (nvec <= 512) quantize_rows_kernel<16, I8><<<grid, block, 0, s>>>(x, rows, cols, ld_x, clip, codes, scales);
  else quantize_rows_long_kernel<I8><<<grid, block, 0, s>>>(x, rows, cols, ld_x, clip, codes, scales);
  return cudaGetLastError();
}

cudaError_t launch_quantize_rows(const __half* x, int64_t rows, int cols, int64_t ld_x, float clip,
                                 uint8_t* codes, float* scales, cudaStream_t s) {
  return launch_quantize_impl<false>(x, rows, cols, ld_x, clip, codes, scales, s);
}
cudaError_t launch_quantize_rows_i8(const __half* x, int64_t rows, int cols, int64_t ld_x, float clip,
                                    int8_t* codes, float* scales, cudaStream_t s) {
  return launch_quantize_impl<true>(x, rows, cols, ld_x, clip, reinterpret_cast<uint8_t*>(codes), scales, s);
}

// Empty kernel with the encoder's launch attributes (q4_launch_floor, measurement only): the
// same prologue handshake as the hot kernels (launch_dependents, then wait) and nothing else.
__global__ void floor_kernel() {
  pdl_launch_dependents();
  pdl_wait();
}
cudaError_t launch_floor_kernel(int ctas, cudaStream_t s) {
  note_launch();
  return launch_pdl(true, floor_kernel, dim3(ctas), dim3(128), 0, s);
}

}  // namespace q4

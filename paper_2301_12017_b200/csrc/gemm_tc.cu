// gemm_tc.cu -- a3..a6: W4A4 linear on the 5th-gen tensor cores (sm_100a).
//
//   acc[m,n] = sum_k qa[m,k] qw[n,k]   exact INT32
//   + fused epilogue: dequant x token scale x channel scale + bias,
//     then GELU+requant or residual+LayerNorm+requant.
//
// B200 has no INT4 tensor datapath, so INT4 is the HBM/L2 storage format
// and the contraction runs as tcgen05.mma kind::i8:
//   warp 0      TMA producer: packed A [128 x BK/2 B] and B [TN x BK/2 B] tiles -> smem ring
//   warps 2..5  unpack: nibbles -> int8 "16*q" in the UMMA K-major swizzled layout
//               (K-permutation trick: lo = (w<<4)&0xF0F0F0F0,
//               hi = w&0xF0F0F0F0, the same permutation of k for A and B, so the
//               INT32 sum is exactly 256 * sum(qa*qw))
//   warp 1      one elected thread issues tcgen05.mma kind::i8 (M=128, N<=256, K=32)
//               into a TMEM accumulator; tcgen05.commit frees smem stages
//   warps 2..5  epilogue: tcgen05.ld thread-per-row, acc>>8 folded into the scale.
// Row epilogues (GELU_Q4 / RESLN_Q4) need the whole output row: the N-tiles of one
// 128-row block form a thread-block cluster and exchange per-row partial statistics
// (shifted moments for LayerNorm, max-abs for the requant scale) through DSMEM.
#include <cstdio>
#include <mutex>

#include "kernels.h"

namespace q4 {

enum { EPI_I32 = 0, EPI_F16 = 1, EPI_GELU_Q4 = 2, EPI_RESLN_Q4 = 3 };

struct TcParams {
  int M, N, K;
  int cluster_n;
  const float* a_scales;
  const float* w_scales;
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

template <int TN, int BK>
struct TcCfg {
  static constexpr int BM = 128;
  static constexpr int PITCH = BK;       // unpacked int8 row bytes
  static constexpr int PPITCH = BK / 2;  // packed row bytes
  static constexpr uint32_t LAYOUT = BK == 128 ? 2u : 4u;  // SWIZZLE_128B / SWIZZLE_64B
  static constexpr int SBO = 8 * PITCH;
  static constexpr int SP = BK == 128 ? 3 : 4;  // packed stages
  static constexpr int SU = 2;                  // unpacked stages
  static constexpr int NMMA = TN > 256 ? 256 : TN;
  static constexpr int NSUB = TN / NMMA;
  static constexpr int A_PK = BM * PPITCH, B_PK = TN * PPITCH;
  static constexpr int A_UN = BM * PITCH, B_UN = TN * PITCH;
  static constexpr int UN_STAGE = A_UN + B_UN;
  static constexpr int PK_STAGE = A_PK + B_PK;
  static constexpr int OFF_UN = 0;
  static constexpr int OFF_PK = SU * UN_STAGE;
  static constexpr int OFF_BAR = OFF_PK + SP * PK_STAGE;
  static constexpr int OFF_X1 = OFF_BAR + 256;          // [16][128] float2 (mean, M2)
  static constexpr int OFF_X2 = OFF_X1 + 16 * 128 * 8;  // [16][128] float  (amax)
  static constexpr int SMEM = OFF_X2 + 16 * 128 * 4 + 1024;
  static constexpr int TMEM_COLS = TN <= 32 ? 32 : TN <= 64 ? 64 : TN <= 128 ? 128 : TN <= 256 ? 256 : 512;
  static constexpr int CPR = BK / 32;  // 16-byte packed chunks per row per k-block
  static_assert(TN % 16 == 0 && (TN <= 256 || TN % 256 == 0), "tile N");
  static_assert(SMEM <= 227 * 1024, "smem");
};

// Physical 16-byte chunk of logical chunk c in row r of a swizzled K-major tile.
template <int BK>
Q4_DEV uint32_t swz(uint32_t r, uint32_t c) {
  if constexpr (BK == 128) return c ^ (r & 7u);
  else return c ^ ((r >> 1) & 3u);
}

// Unpack `rows` x BK/2 packed bytes into rows x BK int8 (16*q), swizzled.
template <int BK>
Q4_DEV void unpack_tile(const uint8_t* __restrict__ pk, uint8_t* __restrict__ un, int rows, int t) {
  constexpr int CPR = BK / 32;
  const int n = rows * CPR;
  for (int i = t; i < n; i += 128) {
    const uint32_t r = (uint32_t)i / CPR, c = (uint32_t)i % CPR;
    const uint4 w = *reinterpret_cast<const uint4*>(pk + (size_t)i * 16);
    uint4 lo, hi;
    lo.x = nib_lo16(w.x); lo.y = nib_lo16(w.y); lo.z = nib_lo16(w.z); lo.w = nib_lo16(w.w);
    hi.x = nib_hi16(w.x); hi.y = nib_hi16(w.y); hi.z = nib_hi16(w.z); hi.w = nib_hi16(w.w);
    uint8_t* row = un + (size_t)r * BK;
    *reinterpret_cast<uint4*>(row + swz<BK>(r, 2 * c) * 16) = lo;
    *reinterpret_cast<uint4*>(row + swz<BK>(r, 2 * c + 1) * 16) = hi;
  }
}

template <int TN, int BK, int KIND>
__global__ void __launch_bounds__(192, 1)
    w4a4_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const TcParams p) {
  using C = TcCfg<TN, BK>;
  constexpr bool ROW = (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full_p = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty_p = full_p + C::SP;
  uint64_t* full_u = empty_p + C::SP;
  uint64_t* empty_u = full_u + C::SU;
  uint64_t* tmem_full = empty_u + C::SU;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float2* x1 = reinterpret_cast<float2*>(smem + C::OFF_X1);
  float* x2 = reinterpret_cast<float*>(smem + C::OFF_X2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * TN;
  const int m0 = blockIdx.y * C::BM;
  const int KB = (p.K + BK - 1) / BK;
  const uint32_t rank = ROW ? cluster_ctarank() : 0u;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::SP; ++i) { mbar_init(&full_p[i], 1); mbar_init(&empty_p[i], 4); }
    for (int i = 0; i < C::SU; ++i) { mbar_init(&full_u[i], 4); mbar_init(&empty_u[i], 1); }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (ROW) cluster_sync();  // every CTA of the cluster is resident before DSMEM use

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % C::SP;
        const uint32_t ph = (uint32_t)(kb / C::SP) & 1u;
        mbar_wait(&empty_p[s], ph ^ 1u);
        uint8_t* pk = smem + C::OFF_PK + s * C::PK_STAGE;
        mbar_arrive_expect_tx(&full_p[s], (uint32_t)C::PK_STAGE);
        tma_load_2d(pk, &tmA, &full_p[s], kb * C::PPITCH, m0);
#pragma unroll
        for (int sub = 0; sub < C::NSUB; ++sub)
          tma_load_2d(pk + C::A_PK + sub * C::NMMA * C::PPITCH, &tmB, &full_p[s], kb * C::PPITCH,
                      n0 + sub * C::NMMA);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_i8(128, C::NMMA);
      for (int kb = 0; kb < KB; ++kb) {
        const int su = kb % C::SU;
        const uint32_t ph = (uint32_t)(kb / C::SU) & 1u;
        mbar_wait(&full_u[su], ph);
        tc_fence_after();
        const uint32_t ua = smem_u32(smem + C::OFF_UN + su * C::UN_STAGE);
        const uint32_t ub = ua + C::A_UN;
#pragma unroll
        for (int ks = 0; ks < BK / 32; ++ks) {
#pragma unroll
          for (int sub = 0; sub < C::NSUB; ++sub) {
            const uint64_t ad = umma_smem_desc(ua + ks * 32, C::SBO, C::LAYOUT);
            const uint64_t bd = umma_smem_desc(ub + sub * C::NMMA * C::PITCH + ks * 32, C::SBO, C::LAYOUT);
            umma_i8(tmem + sub * C::NMMA, ad, bd, idesc, (kb | ks) != 0);
          }
        }
        umma_commit(&empty_u[su]);
      }
      umma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- unpack
    const int t = threadIdx.x - 64;
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % C::SP, su = kb % C::SU;
      mbar_wait(&full_p[s], (uint32_t)(kb / C::SP) & 1u);
      mbar_wait(&empty_u[su], ((uint32_t)(kb / C::SU) & 1u) ^ 1u);
      const uint8_t* pk = smem + C::OFF_PK + s * C::PK_STAGE;
      uint8_t* un = smem + C::OFF_UN + su * C::UN_STAGE;
      unpack_tile<BK>(pk, un, C::BM, t);
      unpack_tile<BK>(pk + C::A_PK, un + C::A_UN, TN, t);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&full_u[su]);
        mbar_arrive(&empty_p[s]);
      }
    }
  }

  // ------------------------------------------------------------------ epilogue
  const bool epi = warp >= 2;
  const int q = warp & 3;
  const int r = q * 32 + lane;  // row within the tile == TMEM lane
  const int gm = m0 + r;
  const bool row_ok = epi && gm < p.M;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int N = p.N;
  float sa = 0.f;
  if (epi) {
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    sa = row_ok ? p.a_scales[gm] * (1.0f / 256.0f) : 0.f;
  }

  if constexpr (KIND == EPI_I32) {
    if (epi) {
      for (int c = 0; c < TN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        tmem_wait_ld();
        if (row_ok) {
          int4* o = reinterpret_cast<int4*>(p.out_i32 + (size_t)gm * N + n0 + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            o[j] = make_int4((int)v[4 * j] >> 8, (int)v[4 * j + 1] >> 8, (int)v[4 * j + 2] >> 8,
                             (int)v[4 * j + 3] >> 8);
        }
      }
    }
  } else if constexpr (KIND == EPI_F16) {
    if (epi) {
      for (int c = 0; c < TN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        tmem_wait_ld();
        const int nb = n0 + c * 32;
        uint32_t h[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = nb + 2 * j;
          const float b0 = p.bias ? __half2float(p.bias[n]) : 0.f;
          const float b1 = p.bias ? __half2float(p.bias[n + 1]) : 0.f;
          const float t0 = fmaf((float)(int)v[2 * j] * sa, __ldg(p.w_scales + n), b0);
          const float t1 = fmaf((float)(int)v[2 * j + 1] * sa, __ldg(p.w_scales + n + 1), b1);
          h[j] = pack_half2(t0, t1);
        }
        if (row_ok) {
          uint4* o = reinterpret_cast<uint4*>(p.out_f16 + (size_t)gm * N + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = make_uint4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- row epilogues
    const int CN = p.cluster_n;
    const float clip = p.clip;
    float mean = 0.f, rstd = 0.f;
    if constexpr (KIND == EPI_RESLN_Q4) {
      // pass 1: z = t + residual, shifted moments, z -> TMEM (in place)
      if (epi) {
        float piv = 0.f, s1 = 0.f, s2 = 0.f;
        for (int c = 0; c < TN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(trow + c * 32, v);
          const int nb = n0 + c * 32;
          uint4 rr[4] = {};
          if (row_ok) {
            const uint4* rp = reinterpret_cast<const uint4*>(p.residual + (size_t)gm * N + nb);
#pragma unroll
            for (int j = 0; j < 4; ++j) rr[j] = __ldg(rp + j);
          }
          const uint32_t* ru = reinterpret_cast<const uint32_t*>(rr);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = nb + 2 * j;
            const float2 res = unpack_half2(ru[j]);
            const float b0 = p.bias ? __half2float(p.bias[n]) : 0.f;
            const float b1 = p.bias ? __half2float(p.bias[n + 1]) : 0.f;
            const float z0 = fmaf((float)(int)v[2 * j] * sa, __ldg(p.w_scales + n), b0) + res.x;
            const float z1 = fmaf((float)(int)v[2 * j + 1] * sa, __ldg(p.w_scales + n + 1), b1) + res.y;
            if (c == 0 && j == 0) piv = z0;
            const float d0 = z0 - piv, d1 = z1 - piv;
            s1 += d0 + d1;
            s2 = fmaf(d0, d0, fmaf(d1, d1, s2));
            v[2 * j] = __float_as_uint(z0);
            v[2 * j + 1] = __float_as_uint(z1);
          }
          tmem_st32(trow + c * 32, v);
        }
        tmem_wait_st();
        const float inv_n = 1.0f / (float)TN;
        const float lmean = piv + s1 * inv_n;
        const float lm2 = fmaxf(s2 - s1 * s1 * inv_n, 0.f);
        const uint32_t la = smem_u32(&x1[rank * 128 + r]);
        for (int k = 0; k < CN; ++k) st_cluster_v2f32(mapa(la, (uint32_t)k), lmean, lm2);
      }
      __syncwarp();
      cluster_sync();
      if (epi) {
        // Chan et al. pairwise combination, in rank order (identical on every CTA)
        float2 s = x1[r];
        float cnt = (float)TN;
        mean = s.x;
        float m2 = s.y;
        for (int k = 1; k < CN; ++k) {
          const float2 o = x1[k * 128 + r];
          const float tot = cnt + (float)TN;
          const float d = o.x - mean;
          mean = fmaf(d, (float)TN / tot, mean);
          m2 = m2 + o.y + d * d * (cnt * (float)TN / tot);
          cnt = tot;
        }
        rstd = 1.0f / sqrtf(m2 / cnt + p.ln_eps);
      }
    }
    // pass A: final fp16 values y (GELU or LN), row max-abs, y -> TMEM as packed halves
    float amax = 0.f;
    if (epi) {
      for (int c = 0; c < TN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        tmem_wait_ld();
        const int nb = n0 + c * 32;
        uint32_t h[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = nb + 2 * j;
          float y0, y1;
          if constexpr (KIND == EPI_RESLN_Q4) {
            y0 = fmaf((__uint_as_float(v[2 * j]) - mean) * rstd, __half2float(p.gamma[n]), __half2float(p.beta[n]));
            y1 = fmaf((__uint_as_float(v[2 * j + 1]) - mean) * rstd, __half2float(p.gamma[n + 1]), __half2float(p.beta[n + 1]));
          } else {
            const float b0 = p.bias ? __half2float(p.bias[n]) : 0.f;
            const float b1 = p.bias ? __half2float(p.bias[n + 1]) : 0.f;
            y0 = gelu_erf(fmaf((float)(int)v[2 * j] * sa, __ldg(p.w_scales + n), b0));
            y1 = gelu_erf(fmaf((float)(int)v[2 * j + 1] * sa, __ldg(p.w_scales + n + 1), b1));
          }
          h[j] = pack_half2(y0, y1);
          float2 f = unpack_half2(h[j]);
          if (clip > 0.f) {
            f.x = fminf(fmaxf(f.x, -clip), clip);
            f.y = fminf(fmaxf(f.y, -clip), clip);
          }
          amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
        if (row_ok && p.out_f16) {
          uint4* o = reinterpret_cast<uint4*>(p.out_f16 + (size_t)gm * N + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = make_uint4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
        }
        tmem_st16(trow + c * 32, h);
      }
      tmem_wait_st();
      const uint32_t la = smem_u32(&x2[rank * 128 + r]);
      for (int k = 0; k < CN; ++k) st_cluster_f32(mapa(la, (uint32_t)k), amax);
    }
    __syncwarp();
    cluster_sync();
    if (epi) {
      amax = x2[r];
      for (int k = 1; k < CN; ++k) amax = fmaxf(amax, x2[k * 128 + r]);
      // pass B: codes = rint(div.rn(7y, amax)), packed (R1-R3)
      for (int c = 0; c < TN / 32; ++c) {
        uint32_t h[16];
        tmem_ld16(trow + c * 32, h);
        tmem_wait_ld();
        uint32_t w[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          int qv[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 f = unpack_half2(h[4 * g + j]);
            if (clip > 0.f) {
              f.x = fminf(fmaxf(f.x, -clip), clip);
              f.y = fminf(fmaxf(f.y, -clip), clip);
            }
            qv[2 * j] = amax > 0.f ? q4_code(f.x, amax) : 0;
            qv[2 * j + 1] = amax > 0.f ? q4_code(f.y, amax) : 0;
          }
          w[g] = pack8(qv);
        }
        if (row_ok)
          *reinterpret_cast<uint4*>(p.out_codes + (size_t)gm * (N / 2) + (n0 + c * 32) / 2) =
              make_uint4(w[0], w[1], w[2], w[3]);
      }
      if (row_ok && rank == 0) p.out_scales[gm] = amax > 0.f ? __fdiv_rn(amax, 7.0f) : 1.0f;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// ====================================================================== host side

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D uint8 tensor map over a row-major [rows, row_bytes] buffer, box [box_rows, box_bytes].
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t row_bytes,
               uint32_t box_rows, uint32_t box_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int TN, int BK, int KIND>
cudaError_t run_tc(const GemmArgs& g, int cluster_n, cudaStream_t s, const char** why) {
  using C = TcCfg<TN, BK>;
  auto kern = w4a4_tc_kernel<TN, BK, KIND>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap ta, tb;
  const uint64_t kb = (uint64_t)g.K / 2;
  if (!make_tmap(&ta, g.a_codes, (uint64_t)g.M, kb, 128, C::PPITCH) ||
      !make_tmap(&tb, g.w_codes, (uint64_t)g.N, kb, C::NMMA, C::PPITCH)) {
    *why = "cuTensorMapEncodeTiled failed (driver entry point or alignment)";
    return cudaErrorInvalidValue;
  }
  TcParams p;
  p.M = g.M; p.N = g.N; p.K = g.K; p.cluster_n = cluster_n;
  p.a_scales = g.a_scales; p.w_scales = g.w_scales;
  p.bias = g.bias; p.residual = g.residual; p.gamma = g.gamma; p.beta = g.beta;
  p.ln_eps = g.ln_eps; p.clip = g.clip;
  p.out_i32 = g.out_i32; p.out_f16 = g.out_f16; p.out_codes = g.out_codes; p.out_scales = g.out_scales;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(g.N / TN), (unsigned)((g.M + 127) / 128), 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cluster_n;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
}

template <int TN, int BK>
cudaError_t run_tc_kind(const GemmArgs& g, int cluster_n, cudaStream_t s, const char** why) {
  switch (g.kind) {
    case EPI_I32: return run_tc<TN, BK, EPI_I32>(g, cluster_n, s, why);
    case EPI_F16: return run_tc<TN, BK, EPI_F16>(g, cluster_n, s, why);
    case EPI_GELU_Q4: return run_tc<TN, BK, EPI_GELU_Q4>(g, cluster_n, s, why);
    case EPI_RESLN_Q4: return run_tc<TN, BK, EPI_RESLN_Q4>(g, cluster_n, s, why);
  }
  *why = "unknown epilogue kind";
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_w4a4_tc(const GemmArgs& g, cudaStream_t s, const char** why) {
  if (g.M == 0) return cudaSuccess;
  const bool row = g.kind == EPI_GELU_Q4 || g.kind == EPI_RESLN_Q4;
  // Tile N: the largest instantiated width dividing N.  Row epilogues put all N-tiles
  // of a row block in one cluster (<= 16 CTAs), so they prefer wide tiles.
  static const int cand[] = {512, 256, 192, 128, 64, 32};
  int tn = 0;
  for (int c : cand) {
    if (g.N % c) continue;
    if (c == 512 && (!row || g.N <= 2048)) continue;  // 512 only to keep clusters <= 8
    tn = c;
    break;
  }
  if (!tn) { *why = "N must be a multiple of 32"; return cudaErrorNotSupported; }
  const int cn = row ? g.N / tn : 1;
  if (cn > 16) { *why = "row epilogues (GELU_Q4 / RESLN_Q4) need N <= 4096 on this path"; return cudaErrorNotSupported; }
  switch (tn) {
    case 512: return run_tc_kind<512, 64>(g, cn, s, why);
    case 256: return run_tc_kind<256, 128>(g, cn, s, why);
    case 192: return run_tc_kind<192, 128>(g, cn, s, why);
    case 128: return run_tc_kind<128, 128>(g, cn, s, why);
    case 64: return run_tc_kind<64, 128>(g, cn, s, why);
    default: return run_tc_kind<32, 128>(g, cn, s, why);
  }
}

}  // namespace q4

// gemm_sparse.cu -- SURVEY 8(f) NEXT-4: W4A4 linear with 2:4-sparse weights ("Pair-(2:4)",
// l1-pruned, then quantized) on the sparse tensor cores
// (tcgen05.mma.sp.cta_group::1.kind::i8).
//
// The sparse operand of tcgen05.mma.sp is A, so the product is computed transposed:
//   D[n, m] = sum_k W[n, k] X[m, k]      (TMEM lane = output channel n, column = token m)
// A = the weight tile [128 channels x 256 logical K] compressed to its two kept values per
//     group of four (int8 16*q, 128 bytes per row, SWIZZLE_128B, straight from HBM by TMA);
//     the 2-bit positions (one nibble i0 | i1 << 2 per group, groups in K order, 8 per 32-bit
//     word) live in TMEM: two columns per MMA (64 logical K), staged once per CTA because the
//     CTA's channel block is fixed (q4_sparse24_compress writes exactly this layout; verified
//     by scripts/probes/umma_sp.cu).
// B = the activation tile [128 tokens x 256 K]: packed INT4 codes TMA'd, unpacked on chip to
//     int8 16*q in NATURAL K order (the 2:4 groups are four consecutive k; the dense kernel's
//     even/odd K permutation would split them), as two SWIZZLE_128B tiles of 128 K.
// Epilogue (thread = channel): F16 t = acc sa[m] sw[n] + b[n] or I32, transposed to the
// row-major [M, N] output through a per-warp shared-memory block.
// Persistent CTA per SM: CTA (g, nb) owns channel block nb and walks token blocks g, g + groups.
#include <cstdio>
#include <mutex>

#include "../../include/q4.h"
#include "kernels.h"

namespace q4 {
namespace {

constexpr int SP_TM = 128, SP_TT = 128, SP_KB = 256;   // channels, tokens, logical K per stage
constexpr int SP_A = SP_TM * 128;                       // compressed weights: 128 rows x 128 B
constexpr int SP_B = 2 * SP_TT * 128;                   // unpacked tokens: two 128 x 128 B tiles
constexpr int SP_PK = SP_TT * 128;                      // packed tokens: 128 rows x 128 B (256 nibbles)
constexpr int SP_SU = 3, SP_SP = 3;                     // unpacked / packed stages
constexpr int SP_UN = SP_A + SP_B;
constexpr int SP_OFF_PK = SP_SU * SP_UN;
constexpr int SP_OFF_STG = SP_OFF_PK + SP_SP * SP_PK;  // 8 epilogue warps x 4 KB transpose blocks
constexpr int SP_OFF_SA = SP_OFF_STG + 8 * 4096;        // [2 groups][128] token scales
constexpr int SP_OFF_BAR = SP_OFF_SA + 2 * 128 * 4;
constexpr int SP_SMEM = SP_OFF_BAR + 256 + 1024;
constexpr int SP_THREADS = (8 + 4 + 2) * 32;            // 2 x 4 epilogue, 4 unpack, producer, MMA
static_assert(SP_SMEM <= 227 * 1024, "smem");

struct SpParams {
  int M, N, K, ntn, mblocks, groups;
  const float* a_scales;
  const float* w_scales;
  const __half* bias;
  const uint32_t* meta;  // [N][K/32] metadata words
  int32_t* out_i32;
  __half* out_f16;
};

// 32 packed nibbles (k0..k31 of one row, k0 in the low nibble) -> 32 int8 16*q in K order
Q4_DEV void unpack_natural(uint4 w, uint4& o0, uint4& o1) {
  const uint32_t in[4] = {w.x, w.y, w.z, w.w};
  uint32_t o[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = (in[i] << 4) & 0xF0F0F0F0u, hi = in[i] & 0xF0F0F0F0u;  // 16 q of even / odd k
    o[2 * i] = prmt(lo, hi, 0x5140u);      // k 0, 1, 2, 3 of this word
    o[2 * i + 1] = prmt(lo, hi, 0x7362u);  // k 4, 5, 6, 7
  }
  o0 = make_uint4(o[0], o[1], o[2], o[3]);
  o1 = make_uint4(o[4], o[5], o[6], o[7]);
}

Q4_DEV void umma_sp_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t e, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %5, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(e),
      "r"(acc), "r"(idesc)
      : "memory");
}
Q4_DEV void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
Q4_DEV void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int KIND>
__global__ void __launch_bounds__(SP_THREADS, 1)
    w4a4_sparse24_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                         const SpParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full_p = reinterpret_cast<uint64_t*>(smem + SP_OFF_BAR);
  uint64_t* empty_p = full_p + SP_SP;
  uint64_t* full_u = empty_p + SP_SP;
  uint64_t* empty_u = full_u + SP_SU;
  uint64_t* tfull = empty_u + SP_SU;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int WU = 8, WP = 12, WM = 13;
  const int KB = p.K / SP_KB;
  const int rank = blockIdx.x % p.ntn;     // this CTA's channel block
  const int g0 = blockIdx.x / p.ntn;       // first token block
  if (warp == WP && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < SP_SP; ++i) { mbar_init(&full_p[i], 1); mbar_init(&empty_p[i], 4); }
    for (int i = 0; i < SP_SU; ++i) { mbar_init(&full_u[i], 5); mbar_init(&empty_u[i], 1); }  // 4 unpack warps + expect_tx
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    fence_mbar_init();
  }
  if (warp == WM) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();
  // metadata of this CTA's 128 channels x K -> TMEM columns [256, 256 + K/32): lane = channel
  if (warp < 4) {
    const int ch = rank * SP_TM + 32 * warp + lane;
    const uint32_t* mr = p.meta + (size_t)ch * (p.K / 32);
    for (int c = 0; c < p.K / 32; c += 8) {
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldg(mr + c + i);
      tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + 256 + c, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == WP) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t g = 0;
      for (int mb = g0; mb < p.mblocks; mb += p.groups) {
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % SP_SP, su = g % SP_SU;
          mbar_wait(&empty_p[s], ((g / SP_SP) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full_p[s], (uint32_t)SP_PK);
          tma_load_2d(smem + SP_OFF_PK + s * SP_PK, &tmX, &full_p[s], kb * 128, mb * SP_TT);
          mbar_wait(&empty_u[su], ((g / SP_SU) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full_u[su], (uint32_t)SP_A);
          tma_load_2d(smem + su * SP_UN, &tmW, &full_u[su], kb * 128, rank * SP_TM);
        }
      }
    }
    __syncwarp();
  } else if (warp == WM) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_i8(SP_TM, SP_TT) | (1u << 2);  // sparse A
      uint32_t g = 0, tcount = 0;
      for (int mb = g0; mb < p.mblocks; mb += p.groups, ++tcount) {
        const uint32_t b = tcount & 1u;
        mbar_wait(&tempty[b], ((tcount >> 1) & 1u) ^ 1u);
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int su = g % SP_SU;
          mbar_wait(&full_u[su], (g / SP_SU) & 1u);
          tc_fence_after();
          const uint32_t ua = smem_u32(smem + su * SP_UN), ub = ua + SP_A;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // 64 logical K per MMA: 32 compressed bytes of A, 64 of B
            umma_sp_i8(tmem + b * SP_TT, umma_smem_desc(ua + ks * 32, 1024, 2),
                       umma_smem_desc(ub + (ks >> 1) * (SP_TT * 128) + (ks & 1) * 64, 1024, 2),
                       tmem + 256 + 2 * (kb * 4 + ks), idesc, (kb | ks) != 0);
          umma_commit(&empty_u[su]);
        }
        umma_commit(&tfull[b]);
      }
    }
    __syncwarp();
  } else if (warp >= WU) {
    // ------------------------------------------------------------ unpack (natural K order)
    const int t = threadIdx.x - 32 * WU;
    const int c = t & 7;  // 16-byte packed chunk = logical K 32c .. 32c + 31 of the stage
    uint32_t g = 0;
    for (int mb = g0; mb < p.mblocks; mb += p.groups) {
      for (int kb = 0; kb < KB; ++kb, ++g) {
        const int s = g % SP_SP, su = g % SP_SU;
        mbar_wait(&full_p[s], (g / SP_SP) & 1u);
        mbar_wait(&empty_u[su], ((g / SP_SU) & 1u) ^ 1u);
        const uint8_t* pk = smem + SP_OFF_PK + s * SP_PK;
        uint8_t* un = smem + su * SP_UN + SP_A + (c >> 2) * (SP_TT * 128);  // tile of this chunk's K
        const uint32_t oc = (uint32_t)(2 * c) & 7u;                         // first output chunk in the tile
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = (t >> 3) + 16 * j;
          uint4 o0, o1;
          unpack_natural(*reinterpret_cast<const uint4*>(pk + r * 128 + c * 16), o0, o1);
          const uint32_t key = (uint32_t)r & 7u;
          *reinterpret_cast<uint4*>(un + r * 128 + ((oc ^ key) << 4)) = o0;
          *reinterpret_cast<uint4*>(un + r * 128 + (((oc + 1) ^ key) << 4)) = o1;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full_u[su]);
          mbar_arrive(&empty_p[s]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (thread = channel)
    const int grp = warp >> 2, q = warp & 3;
    const int n = rank * SP_TM + 32 * q + lane;  // this thread's output channel
    const float sw = p.w_scales[n];
    const float bn = p.bias ? __half2float(p.bias[n]) : 0.f;
    float* sa_s = reinterpret_cast<float*>(smem + SP_OFF_SA) + grp * 128;
    uint8_t* blk = smem + SP_OFF_STG + warp * 4096;  // 32 tokens x 32 channels (x 4 B max)
    uint32_t tcount = 0;
    for (int mb = g0; mb < p.mblocks; mb += p.groups, ++tcount) {
      const uint32_t b = tcount & 1u;
      if ((int)b != grp) continue;
      const int m0 = mb * SP_TT;
      {
        const int m = m0 + 32 * q + lane;
        sa_s[32 * q + lane] = m < p.M ? p.a_scales[m] * (1.0f / 256.0f) : 0.f;  // 16 q x 16 q
      }
      if (q == 0) mbar_wait(&tfull[b], (tcount >> 1) & 1u);
      nbar(1 + grp, 128);
      tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(32 * q) << 16) + b * SP_TT;
      for (int j = 0; j < SP_TT / 32; ++j) {  // 32 tokens per chunk
        uint32_t v[32];
        tmem_ld32(tb + 32 * j, v);
        tmem_wait_ld();
        if constexpr (KIND == 0) {  // I32: acc = 256 x sum qa qw
#pragma unroll
          for (int i = 0; i < 32; ++i) reinterpret_cast<int32_t*>(blk)[i * 32 + lane] = (int)v[i] >> 8;
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            reinterpret_cast<__half*>(blk)[i * 32 + lane] =
                __float2half_rn(fmaf((float)(int)v[i] * sa_s[32 * j + i], sw, bn));
        }
        __syncwarp();
        // block row i = token m0 + 32 j + i: 32 channels contiguous in the [M, N] output
        constexpr int EB = KIND == 0 ? 4 : 2, RB = 32 * EB / 16;  // 16-byte chunks per block row
        for (int idx = lane; idx < 32 * RB; idx += 32) {
          const int i = idx / RB, cc = idx % RB, m = m0 + 32 * j + i;
          if (m < p.M) {
            const uint4 x = *reinterpret_cast<const uint4*>(blk + i * 32 * EB + cc * 16);
            uint8_t* dst = reinterpret_cast<uint8_t*>(KIND == 0 ? (void*)p.out_i32 : (void*)p.out_f16) +
                           ((size_t)m * p.N + rank * SP_TM + 32 * q) * EB + cc * 16;
            *reinterpret_cast<uint4*>(dst) = x;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      nbar(1 + grp, 128);  // sa_s of this group is rewritten by its next tile
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WM) tmem_dealloc(tmem, 512);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool sp_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t row_bytes, bool swz) {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(q);
  });
  if (!fn) return false;
  cuuint64_t dims[2] = {row_bytes, rows}, strides[1] = {row_bytes};
  cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int KIND>
cudaError_t run_sparse(const SparseArgs& a, cudaStream_t s, const char** why) {
  auto kern = w4a4_sparse24_kernel<KIND>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SP_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap tw, tx;
  if (!sp_tmap(&tw, a.w_vals, (uint64_t)a.N, (uint64_t)a.K / 2, true) ||
      !sp_tmap(&tx, a.a_codes, (uint64_t)a.M, (uint64_t)a.K / 2, false)) {
    *why = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  int sms = 0, d = 0;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
  SpParams p;
  p.M = a.M; p.N = a.N; p.K = a.K;
  p.ntn = a.N / SP_TM;
  p.mblocks = (a.M + SP_TT - 1) / SP_TT;
  if (p.ntn > sms) { *why = "N / 128 exceeds the number of SMs"; return cudaErrorNotSupported; }
  p.groups = sms / p.ntn;
  if (p.groups > p.mblocks) p.groups = p.mblocks;
  p.a_scales = a.a_scales; p.w_scales = a.w_scales; p.bias = a.bias; p.meta = a.w_meta;
  p.out_i32 = a.out_i32; p.out_f16 = a.out_f16;
  note_launch();
  cudaError_t e = launch_pdl(a.M <= kPdlMaxRows, kern, dim3(p.groups * p.ntn), dim3(SP_THREADS), SP_SMEM, s, tw, tx, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// l1 2:4 pruning of fp16 rows along K: in every group of four consecutive
// elements the two largest |w| are kept (ties: the lower index), the other two set to zero.
__global__ void prune24_kernel(const __half* __restrict__ w, __half* __restrict__ out, int64_t groups) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= groups) return;
  const uint2 u = reinterpret_cast<const uint2*>(w)[i];
  __half v[4];
  *reinterpret_cast<uint2*>(v) = u;
  float a[4];
  for (int j = 0; j < 4; ++j) a[j] = fabsf(__half2float(v[j]));
  // rank of element j = number of elements that beat it (larger, or equal with a lower index)
  for (int j = 0; j < 4; ++j) {
    int rk = 0;
    for (int k = 0; k < 4; ++k) rk += (a[k] > a[j]) || (a[k] == a[j] && k < j);
    if (rk >= 2) v[j] = __float2half(0.f);
  }
  reinterpret_cast<uint2*>(out)[i] = *reinterpret_cast<uint2*>(v);
}

// packed 2:4-sparse INT4 codes [N, K/2] -> compressed int8 16*q values [N, K/2] (the two kept
// values of each group of four, in K order) + metadata [N, K/32] words (nibble i0 | i1 << 2 per
// group, 8 groups per word).  A group with fewer than two nonzeros keeps zeros at the lowest free
// positions; more than two nonzeros counts a violation (and is not representable).
__global__ void sparse24_compress_kernel(const uint8_t* __restrict__ codes, int64_t N, int K, int8_t* __restrict__ vals,
                                         uint32_t* __restrict__ meta, int* __restrict__ violations) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one metadata word = 32 K
  const int64_t words = N * (K / 32);
  if (i >= words) return;
  const int64_t n = i / (K / 32), w = i % (K / 32);
  const uint4 u = reinterpret_cast<const uint4*>(codes + n * (K / 2))[w];  // 32 nibbles
  const uint32_t in[4] = {u.x, u.y, u.z, u.w};
  uint32_t mw = 0, ov[4] = {0, 0, 0, 0};
  int bad = 0;
  for (int gq = 0; gq < 8; ++gq) {  // group of 4 nibbles: K 4 gq .. 4 gq + 3
    const uint32_t nib4 = (in[gq >> 1] >> (16 * (gq & 1))) & 0xFFFFu;
    int idx[2] = {-1, -1}, cnt = 0;
    for (int j = 0; j < 4; ++j)
      if ((nib4 >> (4 * j)) & 0xF) {
        if (cnt < 2) idx[cnt] = j;
        ++cnt;
      }
    if (cnt > 2) ++bad;
    if (idx[0] < 0) {  // no nonzero: positions 0, 1 (both zero)
      idx[0] = 0;
      idx[1] = 1;
    } else if (idx[1] < 0) {  // one nonzero: pair it with a zero neighbour, i0 < i1
      if (idx[0] == 3) {
        idx[0] = 2;
        idx[1] = 3;
      } else {
        idx[1] = idx[0] + 1;
      }
    }
    mw |= (uint32_t)(idx[0] | (idx[1] << 2)) << (4 * gq);
    for (int e = 0; e < 2; ++e) {
      const int q = (int)((nib4 >> (4 * idx[e])) & 0xF);
      const int qs = q >= 8 ? q - 16 : q;
      const uint32_t byte = (uint32_t)(uint8_t)(int8_t)(16 * qs);
      const int pos = 2 * gq + e;  // value index within the word's 16 kept values
      ov[pos >> 2] |= byte << (8 * (pos & 3));
    }
  }
  reinterpret_cast<uint4*>(vals + n * (K / 2))[w] = make_uint4(ov[0], ov[1], ov[2], ov[3]);
  meta[i] = mw;
  if (bad && violations) atomicAdd(violations, bad);
}

}  // namespace

cudaError_t launch_w4a4_sparse24(const SparseArgs& a, cudaStream_t s, const char** why) {
  if (a.M == 0) return cudaSuccess;
  return a.out_i32 ? run_sparse<0>(a, s, why) : run_sparse<1>(a, s, why);
}

cudaError_t launch_prune24(const __half* w, int64_t N, int64_t K, __half* out, cudaStream_t s) {
  const int64_t groups = N * K / 4;
  if (groups == 0) return cudaSuccess;
  note_launch();
  prune24_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, s>>>(w, out, groups);
  return cudaGetLastError();
}

cudaError_t launch_sparse24_compress(const uint8_t* codes, int64_t N, int64_t K, int8_t* vals, uint32_t* meta,
                                     int* violations, cudaStream_t s) {
  const int64_t words = N * (K / 32);
  if (words == 0) return cudaSuccess;
  note_launch();
  sparse24_compress_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(codes, N, (int)K, vals, meta, violations);
  return cudaGetLastError();
}

}  // namespace q4

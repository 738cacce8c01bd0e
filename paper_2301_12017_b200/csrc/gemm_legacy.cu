// gemm_legacy.cu -- the Ampere-style W4A4 GEMM the paper's CUTLASS 2.6 kernels map to
// (PAPER.md:410, 420), kept as the measured baseline for the tcgen05 path (north_star:
// "benchmarked against a legacy mma.sync .s4 path and chosen by measurement").
//
//   cp.async 3-stage ring of packed A/B tiles (128 x 64 B each) -> ldmatrix ->
//   S4: mma.sync m16n8k64 .s4.s4   (ptxas lowers it to 2x IMMA.16832.S8 + unpack on sm_100a)
//   S8: register nibble unpack (same K-permutation trick as the tcgen05 path) ->
//       2x mma.sync m16n8k32 .s8.s8, accumulator = 256 * exact, >> 8 in the epilogue.
// CTA tile 128 x 128, 8 warps (2 x 4), warp tile 64 x 32.  Epilogues: I32, F16.
#include "kernels.h"

namespace q4 {

namespace {
constexpr int LBM = 128, LBN = 128, LBK = 128;  // BK in int4 elements = 64 bytes
constexpr int LST = 3;
constexpr int ROWB = LBK / 2;  // 64 bytes per row per k-block

Q4_DEV void cp_async16(uint32_t s, const void* g, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(g), "r"(pred ? 16 : 0) : "memory");
}
// 64-byte rows, 16-byte chunks swizzled so 8 consecutive rows hit 8 distinct bank groups.
Q4_DEV uint32_t loff(int r, int c) { return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4)); }
Q4_DEV void ldsm4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
Q4_DEV void mma_s4(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.s4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
Q4_DEV void mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
}  // namespace

template <bool S4, int KIND>
__global__ void __launch_bounds__(256) w4a4_legacy_kernel(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
                                                          const float* __restrict__ sa, const float* __restrict__ sw,
                                                          const __half* __restrict__ bias, int M, int N, int K,
                                                          int32_t* __restrict__ out_i32, __half* __restrict__ out_f16) {
  __shared__ __align__(128) uint8_t sA[LST][LBM * ROWB];
  __shared__ __align__(128) uint8_t sB[LST][LBN * ROWB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int m0 = blockIdx.y * LBM, n0 = blockIdx.x * LBN;
  const int KB = (K + LBK - 1) / LBK;
  const int kbytes = K / 2;

  auto load = [&](int kb, int st) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * 256;  // 512 chunks per operand (128 rows x 4)
      const int r = idx >> 2, c = idx & 3;
      const int kc = kb * ROWB + c * 16;
      const bool okA = (m0 + r < M) && (kc < kbytes);
      const bool okB = (n0 + r < N) && (kc < kbytes);
      cp_async16(smem_u32(&sA[st][0]) + loff(r, c), A + (size_t)(okA ? m0 + r : 0) * kbytes + (okA ? kc : 0), okA);
      cp_async16(smem_u32(&sB[st][0]) + loff(r, c), B + (size_t)(okB ? n0 + r : 0) * kbytes + (okB ? kc : 0), okB);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0;

  for (int s = 0; s < LST - 1; ++s) {
    if (s < KB) load(s, s);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kb = 0; kb < KB; ++kb) {
    asm volatile("cp.async.wait_group %0;" ::"n"(LST - 2) : "memory");
    __syncthreads();
    const int nk = kb + LST - 1;
    if (nk < KB) load(nk, nk % LST);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const int st = kb % LST;
    const uint32_t a_base = smem_u32(&sA[st][0]), b_base = smem_u32(&sB[st][0]);
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {  // two k64 steps per 64-byte row
      uint32_t af[4][4], bf[2][4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r = wm * 64 + mt * 16 + (lane & 15);
        ldsm4(a_base + loff(r, ks * 2 + (lane >> 4)), af[mt]);
      }
#pragma unroll
      for (int np = 0; np < 2; ++np) {
        const int r = wn * 32 + np * 16 + ((lane >> 4) << 3) + (lane & 7);
        ldsm4(b_base + loff(r, ks * 2 + ((lane >> 3) & 1)), bf[np]);
      }
      if constexpr (S4) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
            mma_s4(acc[mt][nt], af[mt], bf[nt >> 1][(nt & 1) * 2], bf[nt >> 1][(nt & 1) * 2 + 1]);
      } else {
        uint32_t bl[4][2], bh[4][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t w = bf[nt >> 1][(nt & 1) * 2 + h];
            bl[nt][h] = nib_lo16(w);
            bh[nt][h] = nib_hi16(w);
          }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const uint32_t* a = af[mt];
          const uint32_t l0 = nib_lo16(a[0]), l1 = nib_lo16(a[1]), h0 = nib_hi16(a[0]), h1 = nib_hi16(a[1]);
          const uint32_t l2 = nib_lo16(a[2]), l3 = nib_lo16(a[3]), h2 = nib_hi16(a[2]), h3 = nib_hi16(a[3]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            mma_s8(acc[mt][nt], l0, l1, h0, h1, bl[nt][0], bh[nt][0]);
            mma_s8(acc[mt][nt], l2, l3, h2, h3, bl[nt][1], bh[nt][1]);
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  const int g = lane >> 2, t = lane & 3;
  const int shift = S4 ? 0 : 8;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int m = m0 + wm * 64 + mt * 16 + g + hh * 8;
      if (m >= M) continue;
      const float s_a = sa[m];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int n = n0 + wn * 32 + nt * 8 + 2 * t;
        if (n >= N) continue;
        const int v0 = acc[mt][nt][2 * hh] >> shift, v1 = acc[mt][nt][2 * hh + 1] >> shift;
        if constexpr (KIND == 0) {
          *reinterpret_cast<int2*>(out_i32 + (size_t)m * N + n) = make_int2(v0, v1);
        } else {
          const float b0 = bias ? __half2float(bias[n]) : 0.f, b1 = bias ? __half2float(bias[n + 1]) : 0.f;
          const float t0 = fmaf((float)v0 * s_a, sw[n], b0), t1 = fmaf((float)v1 * s_a, sw[n + 1], b1);
          *reinterpret_cast<uint32_t*>(out_f16 + (size_t)m * N + n) = pack_half2(t0, t1);
        }
      }
    }
  }
}

cudaError_t launch_w4a4_legacy(const GemmArgs& g, bool s4, cudaStream_t s, const char** why) {
  if (g.kind != 0 && g.kind != 1) {
    *why = "legacy mma.sync mainloops implement Q4_EPI_I32 and Q4_EPI_F16 only";
    return cudaErrorNotSupported;
  }
  if (g.M == 0) return cudaSuccess;
  const dim3 grid((unsigned)((g.N + LBN - 1) / LBN), (unsigned)((g.M + LBM - 1) / LBM));
  note_launch();
  if (s4) {
    if (g.kind == 0) w4a4_legacy_kernel<true, 0><<<grid, 256, 0, s>>>(g.a_codes, g.w_codes, g.a_scales, g.w_scales, g.bias, g.M, g.N, g.K, g.out_i32, g.out_f16);
    else w4a4_legacy_kernel<true, 1><<<grid, 256, 0, s>>>(g.a_codes, g.w_codes, g.a_scales, g.w_scales, g.bias, g.M, g.N, g.K, g.out_i32, g.out_f16);
  } else {
    if (g.kind == 0) w4a4_legacy_kernel<false, 0><<<grid, 256, 0, s>>>(g.a_codes, g.w_codes, g.a_scales, g.w_scales, g.bias, g.M, g.N, g.K, g.out_i32, g.out_f16);
    else w4a4_legacy_kernel<false, 1><<<grid, 256, 0, s>>>(g.a_codes, g.w_codes, g.a_scales, g.w_scales, g.bias, g.M, g.N, g.K, g.out_i32, g.out_f16);
  }
  return cudaGetLastError();
}

}  // namespace q4

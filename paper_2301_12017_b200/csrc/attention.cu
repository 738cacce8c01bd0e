// attention.cu -- a7: FP16 attention glue between the quantized GEMMs, with the
// per-token INT4 quantize of the context fused in.
//
// At seq <= 128 one tile holds the whole key range, so no online softmax is needed;
// the op is HBM-bound (~64 flop/B vs an fp16 ridge of ~340), so it uses the
// legacy mma.sync m16n8k16 tensor path, FlashAttention-2 style register reuse of P.
//
// CTA = 64 queries of one sequence, 4 warps x 16 rows, looping over all heads with a
// double-buffered cp.async Q/K/V ring (80 KB -> 2 CTAs per SM).  Each warp writes its
// fp16 context rows (coalesced, via a 2 KB smem slab) and keeps the per-token running
// max-abs in registers; after the last head it re-reads its own rows from L2 and writes
// the INT4 codes + scales, so the per-token quantize is fused into the same kernel.
#include "kernels.h"

namespace q4 {

namespace {

constexpr int D = 64;        // head_dim
constexpr int QB = 64;       // queries per CTA
constexpr int SMAX = 128;    // keys per sequence (max)
constexpr int THREADS = 128;

Q4_DEV void cp_async16(void* smem, const void* g, bool pred) {
  const uint32_t s = smem_u32(smem);
  const int n = pred ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(g), "r"(n) : "memory");
}
Q4_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
Q4_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

Q4_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
Q4_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
Q4_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// [rows][64 halves] tile, 16-byte chunks XOR-swizzled by row to keep ldmatrix conflict-free.
Q4_DEV uint32_t tile_off(int row, int chunk) { return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4)); }

struct HeadBuf {
  __half q[QB * D];
  __half k[SMAX * D];
  __half v[SMAX * D];
};
constexpr size_t kSmem = 2 * sizeof(HeadBuf) + 4 * 16 * 128;  // ring + 4 warp slabs (16 rows x 128 B)

}  // namespace

__global__ void __launch_bounds__(THREADS, 2)
    attention_q4_kernel(const __half* __restrict__ qkv, int S, int heads, __half* __restrict__ ctx_f16,
                        uint8_t* __restrict__ ctx_codes, float* __restrict__ ctx_scales) {
  extern __shared__ __align__(128) uint8_t smem[];
  HeadBuf* hb = reinterpret_cast<HeadBuf*>(smem);  // [2]
  const int h = heads * D, ld = 3 * h;
  const int b = blockIdx.y, q0 = blockIdx.x * QB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const __half* base = qkv + (size_t)b * S * ld;
  uint8_t* slab = smem + 2 * sizeof(HeadBuf) + warp * 16 * 128;  // this warp's 16 x 64 fp16 tile

  auto load_head = [&](int j, HeadBuf* dst) {
    for (int i = tid; i < QB * 8; i += THREADS) {
      const int r = i >> 3, c = i & 7;
      const bool ok = q0 + r < S;
      cp_async16(reinterpret_cast<uint8_t*>(dst->q) + tile_off(r, c),
                 base + (size_t)(ok ? q0 + r : 0) * ld + j * D + c * 8, ok);
    }
    for (int i = tid; i < SMAX * 8; i += THREADS) {
      const int r = i >> 3, c = i & 7;
      const bool ok = r < S;
      const __half* src = base + (size_t)(ok ? r : 0) * ld + j * D + c * 8;
      cp_async16(reinterpret_cast<uint8_t*>(dst->k) + tile_off(r, c), src + h, ok);
      cp_async16(reinterpret_cast<uint8_t*>(dst->v) + tile_off(r, c), src + 2 * h, ok);
    }
    cp_async_commit();
  };

  const float sl2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
  const int nkt = (S + 7) / 8;                      // key n-tiles of 8
  float am0 = 0.f, am1 = 0.f;                       // running |ctx| max of rows g, g+8

  load_head(0, &hb[0]);
  for (int j = 0; j < heads; ++j) {
    HeadBuf* cur = &hb[j & 1];
    if (j + 1 < heads) {
      load_head(j + 1, &hb[(j + 1) & 1]);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t sq = smem_u32(cur->q), sk = smem_u32(cur->k), sv = smem_u32(cur->v);

    // Q fragments (16 rows x 64) of this warp
    uint32_t qa[4][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      ldsm_x4(sq + tile_off(warp * 16 + (lane & 15), ks * 2 + (lane >> 4)), qa[ks][0], qa[ks][1],
              qa[ks][2], qa[ks][3]);
    // S = Q K^T
    float sc[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
      if (nt < nkt) {
#pragma unroll
        for (int kp = 0; kp < 2; ++kp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sk + tile_off(nt * 8 + (lane & 7), kp * 4 + (lane >> 3)), b0, b1, b2, b3);
          mma16816(sc[nt], qa[2 * kp], b0, b1);
          mma16816(sc[nt], qa[2 * kp + 1], b2, b3);
        }
      }
    }
    // softmax over the S keys (rows g and g+8 of the warp tile)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int k0 = nt * 8 + 2 * t;
      if (k0 >= S) { sc[nt][0] = sc[nt][2] = -INFINITY; }
      if (k0 + 1 >= S) { sc[nt][1] = sc[nt][3] = -INFINITY; }
      mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    // P = exp(s - max) as A fragments (k-steps of 16 keys), split P = hi + lo with
    // hi = fp16(P), lo = fp16(P - hi): the PV product then carries ~22 bits of P
    // instead of fp16's 11.
    float sum0 = 0.f, sum1 = 0.f;
    uint32_t pa[8][4], pl[8][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const float p0 = exp2f(sc[nt][0] * sl2 - mx0 * sl2);
      const float p1 = exp2f(sc[nt][1] * sl2 - mx0 * sl2);
      const float p2 = exp2f(sc[nt][2] * sl2 - mx1 * sl2);
      const float p3 = exp2f(sc[nt][3] * sl2 - mx1 * sl2);
      sum0 += p0 + p1;
      sum1 += p2 + p3;
      const uint32_t h01 = pack_half2(p0, p1), h23 = pack_half2(p2, p3);
      const float2 f01 = unpack_half2(h01), f23 = unpack_half2(h23);
      pa[nt >> 1][(nt & 1) * 2 + 0] = h01;
      pa[nt >> 1][(nt & 1) * 2 + 1] = h23;
      pl[nt >> 1][(nt & 1) * 2 + 0] = pack_half2(p0 - f01.x, p1 - f01.y);
      pl[nt >> 1][(nt & 1) * 2 + 1] = pack_half2(p2 - f23.x, p3 - f23.y);
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      sum0 += __shfl_xor_sync(0xffffffffu, sum0, o);
      sum1 += __shfl_xor_sync(0xffffffffu, sum1, o);
    }
    // O = P V
    float oc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) oc[nt][0] = oc[nt][1] = oc[nt][2] = oc[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      if (kk * 16 < S) {
#pragma unroll
        for (int np = 0; np < 4; ++np) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sv + tile_off(kk * 16 + (lane & 15), np * 2 + (lane >> 4)), b0, b1, b2, b3);
          mma16816(oc[2 * np], pa[kk], b0, b1);
          mma16816(oc[2 * np + 1], pa[kk], b2, b3);
          mma16816(oc[2 * np], pl[kk], b0, b1);
          mma16816(oc[2 * np + 1], pl[kk], b2, b3);
        }
      }
    }
    const float inv0 = 1.0f / sum0, inv1 = 1.0f / sum1;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const uint32_t h0 = pack_half2(oc[nt][0] * inv0, oc[nt][1] * inv0);
      const uint32_t h1 = pack_half2(oc[nt][2] * inv1, oc[nt][3] * inv1);
      const float2 f0 = unpack_half2(h0), f1 = unpack_half2(h1);
      am0 = fmaxf(am0, fmaxf(fabsf(f0.x), fabsf(f0.y)));
      am1 = fmaxf(am1, fmaxf(fabsf(f1.x), fabsf(f1.y)));
      // slab rows g / g+8; halves nt*8+2t, +1 sit in 16-byte chunk nt at byte 4t
      *reinterpret_cast<uint32_t*>(slab + tile_off(g, nt) + 4 * t) = h0;
      *reinterpret_cast<uint32_t*>(slab + tile_off(g + 8, nt) + 4 * t) = h1;
    }
    __syncwarp();
    // coalesced store of the warp's 16 x 64 ctx tile (4 rows x 128 B per instruction)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = i * 4 + (lane >> 3), ch = lane & 7;
      const int tok = q0 + warp * 16 + rr;
      const uint4 v = *reinterpret_cast<const uint4*>(slab + tile_off(rr, ch));
      if (tok < S) *reinterpret_cast<uint4*>(ctx_f16 + ((size_t)b * S + tok) * h + j * D + ch * 8) = v;
    }
    __syncwarp();
    __syncthreads();  // cur buffer is refilled two heads later
  }

  // per-token max-abs over all heads, then quantize + pack this warp's rows (L2-resident)
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    am0 = fmaxf(am0, __shfl_xor_sync(0xffffffffu, am0, o));
    am1 = fmaxf(am1, __shfl_xor_sync(0xffffffffu, am1, o));
  }
  for (int rr = 0; rr < 16; ++rr) {
    const float a = __shfl_sync(0xffffffffu, (rr & 8) ? am1 : am0, (rr & 7) * 4);
    const int tok = q0 + warp * 16 + rr;
    if (tok >= S) continue;
    const float r7 = a > 0.f ? __fdiv_rn(7.0f, a) : 0.f;
    const size_t grow = (size_t)b * S + tok;
    const uint4* src = reinterpret_cast<const uint4*>(ctx_f16 + grow * h);
    uint32_t* cw = reinterpret_cast<uint32_t*>(ctx_codes + grow * (h / 2));
    uint4 x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < h / 8) x[i] = __ldcg(src + lane + 32 * i);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < h / 8) {
        const uint32_t hh[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
        cw[lane + 32 * i] = requant8(hh, a, r7, 0.f);
      }
    if (lane == 0) ctx_scales[grow] = a > 0.f ? __fdiv_rn(a, 7.0f) : 1.0f;
  }
}

cudaError_t launch_attention(const __half* qkv, int B, int S, int heads, __half* ctx_f16,
                             uint8_t* ctx_codes, float* ctx_scales, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attention_q4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const dim3 grid((unsigned)((S + QB - 1) / QB), (unsigned)B);
  note_launch();
  attention_q4_kernel<<<grid, THREADS, kSmem, s>>>(qkv, S, heads, ctx_f16, ctx_codes, ctx_scales);
  return cudaGetLastError();
}

}  // namespace q4

// attention_tc.cu -- a7 on the 5th-gen tensor cores: FP16 attention + fused per-token
// INT4 quantize of the context.
//
// One CTA per sequence (S <= 128 queries = one MMA M tile), looping over the heads; two
// CTAs per SM (113 KB smem, 256 TMEM columns each) so all 256 sequences of the BERT-large
// batch are resident at once and each CTA's softmax overlaps the other's MMAs/epilogue:
//   warp 8      TMA producer: Q_h, K_h, V_h tiles [128 x 64] fp16 (SWIZZLE_128B) of the
//               QKV activation -> 2-stage smem ring (48 KB per head), L2 evict-first
//   warp 9      MMA issuer:  S_h = Q_h K_h^T   tcgen05.mma kind::f16, M=128 N=128 K=16 (fp32, TMEM)
//                            O_h = P_h V_h     A = P from TMEM (TS form), B = V MN-major smem
//   warps 0-7   TMEM lane quarter q = w & 3 (query rows 32q..32q+31), key half hf = w >> 2:
//               row max / exp2 / row sum of S (halves combined through smem); P = exp split
//               hi + lo fp16 (P = fp16(P) + fp16(P - fp16(P)), ~22 bits) written
//               back over the consumed S columns; then O * (1/sum) -> fp16 ctx (coalesced
//               stores via a smem slab, L2 evict-last) and the per-token running max-abs.
//               After the last head each warp stages 16 of the CTA's rows back from L2 into
//               the idle Q/K/V stages (cp.async) and writes the INT4 codes + scales.
// TMEM: S/P at columns [0,128), O at [128,192), single-buffered (the second CTA on the SM
// provides the overlap a second buffer would).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace q4 {

namespace {

constexpr int AT_THREADS = 320;  // 8 softmax/epilogue warps + producer + MMA
constexpr int NST = 2;                        // Q/K/V ring stages (2 CTAs per SM)
constexpr int TILE = 128 * 128;               // bytes of one [128 x 64] fp16 tile
constexpr int STAGE = 3 * TILE;               // Q | K | V
constexpr int OFF_SLAB = NST * STAGE;         // 8 warps x 16 rows x 64 B
constexpr int OFF_RED = OFF_SLAB + 8 * 1024;  // [2 halves][128] max-abs | asym: [2][128] min | [2][128] max
constexpr int OFF_BAR = OFF_RED + 6 * 128 * 4;
constexpr int SMEM_AT = OFF_BAR + 256 + 1024;
constexpr int kAttnSmemMax = 227 * 1024;  // opt-in ceiling (the launch uses SMEM_AT: two CTAs per SM)

// kind::f16 instruction descriptor: f16 x f16 -> f32, A K-major, B K-major (b_mn = 0) or
// MN-major (b_mn = 1), M x N.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int b_mn) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

Q4_DEV void umma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
Q4_DEV void umma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// fp16 tensor map [rows, cols] row-major, box [128 rows, 64 cols], 128-byte swizzle.
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

// QM: ctx code mode -- 0 symmetric INT4 (a1), 1 int8 (W8A8 baseline, O-11), 2 asymmetric INT4
// (NEXT-3, O-15); one instantiation each, so the hot symmetric kernel carries no other mode.
template <int QM>
__global__ void __launch_bounds__(AT_THREADS, 2)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tq, int S, int heads, __half* __restrict__ ctx_f16,
                        uint8_t* __restrict__ ctx_codes, float* __restrict__ ctx_scales,
                        unsigned long long* __restrict__ trace, int dbg, int G, float* __restrict__ ctx_zeros) {
  constexpr bool i8 = QM == 1, asym = QM == 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* kv_empty = kv_full + NST;
  uint64_t* s_full = kv_empty + NST;
  uint64_t* p_full = s_full + 1;
  uint64_t* o_full = p_full + 1;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = heads * 64;
  // G CTAs (one cluster) per sequence, each running hpc = heads / G consecutive heads
  const int b = blockIdx.x / G, g = blockIdx.x % G;
  const int hpc = heads / G, j0 = g * hpc;
  const int row0 = b * S;  // first token of this sequence
  // profiling only (Q4_TRACE): thread 0's kernel-level stamps in head slot 15 (unused at one
  // head per CTA): [0] kernel entry, [1] after the prologue, [2] tail: first cluster barrier
  // passed, [3] row scales ready, [4] codes written, [5] exit
  auto kstamp = [&](int k) {
    if (trace && threadIdx.x == 0 && blockIdx.x < 512) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      trace[(size_t)blockIdx.x * 256 + 15 * 16 + k] = t;
    }
  };
  kstamp(0);

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tq);
    for (int i = 0; i < NST; ++i) { mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1); }
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 8);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  kstamp(1);
  pdl_launch_dependents();
  pdl_wait();  // everything below may read the previous kernel's outputs
  // TMEM columns: S / P at [0, 128), O at [128, 192) (single-buffered; two CTAs per SM overlap)
  if (warp == 8) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int jj = 0; jj < hpc; ++jj) {
        const int st = jj % NST, j = j0 + jj;
        mbar_wait(&kv_empty[st], ((jj / NST) & 1u) ^ 1u);
        uint8_t* base = smem + st * STAGE;
        mbar_arrive_expect_tx(&kv_full[st], (uint32_t)STAGE);
        // QKV is read once: evict-first keeps L2 for the ctx rows re-read by the quantize
        tma_load_2d_hint(base, &tq, &kv_full[st], j * 64, row0, pol);
        tma_load_2d_hint(base + TILE, &tq, &kv_full[st], h + j * 64, row0, pol);
        tma_load_2d_hint(base + 2 * TILE, &tq, &kv_full[st], 2 * h + j * 64, row0, pol);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_f16(128, 128, 0), idO = idesc_f16(128, 64, 1);
      for (int jj = 0; jj < hpc; ++jj) {
        const int st = jj % NST;
        const uint32_t ph = (uint32_t)jj & 1u;
        mbar_wait(&kv_full[st], (jj / NST) & 1u);
        tc_fence_after();
        const uint32_t q = smem_u32(smem + st * STAGE), k = q + TILE, v = k + TILE;
        // S = Q K^T (in-order after PV of the previous head, which read P from these columns)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)  // K = 64 head dims, 16 per MMA (32 bytes of a 128-byte row)
          umma_f16_ss(tmem, umma_smem_desc(q + ks * 32, 1024, 2), umma_smem_desc(k + ks * 32, 1024, 2), idS, ks != 0);
        umma_commit(s_full);
        mbar_wait(p_full, ph);
        mbar_wait(o_empty, ph ^ 1u);
        tc_fence_after();
        // O = sum over 8 key steps of 16: (P_hi + P_lo)[:, keys] x V[keys, :]
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t vd = umma_smem_desc(v + ks * 2048, 1024, 2);  // 16 keys x 128 B, MN-major
          const uint32_t pc = tmem + 32 * (ks >> 1) + 8 * (ks & 1);
          umma_f16_ts(tmem + 128, pc, vd, idO, ks != 0);
          umma_f16_ts(tmem + 128, pc + 16, vd, idO, 1);
        }
        umma_commit(o_full);
        umma_commit(&kv_empty[st]);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- softmax + epilogue
    // warp w: TMEM lane quarter q = w & 3 (rows 32q..32q+31), half hf = w >> 2 (key columns
    // 64hf..64hf+63 of S / P, output columns 32hf..32hf+31 of O).  Row max / sum / max-abs
    // of the two halves are combined through shared memory.
    const int q = warp & 3, hf = warp >> 2;
    const int r = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const float sl2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
    // ctx rows stay in L2 (evict-last) until the quantize re-reads them (then evict-first)
    const uint64_t pol_keep = l2_policy_evict_last(), pol_drop = l2_policy_evict_first();
    uint8_t* slab = smem + OFF_SLAB + warp * 1024;   // 16 rows x 64 B
    float* red = reinterpret_cast<float*>(smem + OFF_RED);  // [2][128]
    float inv = 0.f;
    float amax = 0.f;
    // asymmetric ctx codes (NEXT-3, ctx_zeros != nullptr): running per-token min and max
    float vmn = INFINITY, vmx = -INFINITY;
    // profiling only (Q4_TRACE): per-head stamps of thread 0 of CTAs < 512
    unsigned long long* tr = (trace && threadIdx.x == 0 && blockIdx.x < 512) ? trace + (size_t)blockIdx.x * 16 * 16 : nullptr;
    auto stamp = [&](int j, int k) {
      if (tr && j < 16) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        tr[j * 16 + k] = t;
      }
    };
    auto combine = [&](float v, bool is_max) {  // both halves of row r
      red[hf * 128 + r] = v;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float o = red[(hf ^ 1) * 128 + r];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      return is_max ? fmaxf(v, o) : v + o;
    };
    // MASKED: the ragged last key block (S - 64 hf < 64); a separate instantiation so the
    // full-tile path carries no per-element selects
    auto softmax = [&](int j, auto masked) {
      stamp(j, 0);
      mbar_wait(s_full, (uint32_t)j & 1u);
      stamp(j, 1);
      tc_fence_after();
      const uint32_t sb = tl + 64 * hf;
      // masked scores -> -inf -> p = 0 (lim = valid key columns in this half)
      auto mask = [&](uint32_t(&v)[32], int c0) {
        if constexpr (decltype(masked)::value) {
          const int lim = S - 64 * hf - c0;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i >= lim) v[i] = 0xFF800000u;
        }
      };
      uint32_t v0[32], v1[32];
      tmem_ld32(sb, v0);
      tmem_ld32(sb + 32, v1);
      tmem_wait_ld();
      mask(v0, 0);
      mask(v1, 32);
      // four independent max chains (latency, not throughput, bounds this loop)
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 32; ++i)
        m4[i & 3] = fmaxf(m4[i & 3], fmaxf(__uint_as_float(v0[i]), __uint_as_float(v1[i])));
      float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      mx = combine(mx, true);
      if (j >= 3) stamp(j, 6);
      const float2 nm2 = f2(-mx * sl2), sl22 = f2(sl2);
      float2 sa = f2(0.f), sb2 = f2(0.f);  // two independent sum chains
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t* v = c ? v1 : v0;
        uint32_t ph[16], pl[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 e = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl22, nm2);
          const float2 pp = make_float2(ex2_approx(e.x), ex2_approx(e.y));
          if (i & 1)
            sb2 = fadd2(sb2, pp);
          else
            sa = fadd2(sa, pp);
          ph[i] = pack_half2(pp.x, pp.y);
          const float2 lo = sub_half2_f32(ph[i], pp);  // exact p - hi
          pl[i] = pack_half2(lo.x, lo.y);
        }
        // P for keys 64 hf + 32 c .. +31 over the consumed S columns: hi at +0, lo at +16
        tmem_st16(sb + 32 * c, ph);
        tmem_st16(sb + 32 * c + 16, pl);
      }
      const float2 sum2 = fadd2(sa, sb2);
      if (j >= 3) stamp(j, 7);
      tmem_wait_st();
      inv = 1.0f / combine(sum2.x + sum2.y, false);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      stamp(j, 2);
    };
    auto epilogue = [&](int j) {
      stamp(j, 3);
      mbar_wait(o_full, (uint32_t)j & 1u);
      stamp(j, 4);
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(tl + 128 + 32 * hf, o);
      tmem_wait_ld();
      stamp(j, 8);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
      const float2 iv2 = f2(inv);
      uint4 hw4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t hw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 y = fmul2(make_float2(__uint_as_float(o[8 * u + 2 * e]), __uint_as_float(o[8 * u + 2 * e + 1])), iv2);
          hw[e] = pack_half2(y.x, y.y);
          // fp16 rounding is monotonic and odd, so max |fp16(y)| == fp16(max |y|) (rounded below)
          amax = fmaxf(amax, fmaxf(fabsf(y.x), fabsf(y.y)));
          if (asym) {  // likewise min / max of fp16(y) == fp16 of the fp32 min / max
            vmn = fminf(vmn, fminf(y.x, y.y));
            vmx = fmaxf(vmx, fmaxf(y.x, y.y));
          }
        }
        hw4[u] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      }
      if (G > 1 && hpc == 1) {
        // one head per CTA: the ctx tile [128 x 64] fp16 also stays in shared memory (the Q/K/V
        // stage is idle once O is complete) for the cluster tail's codes; 16-byte chunk c of row
        // r at c ^ (r & 7)
        uint8_t* ct = smem + r * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(ct + (((hf * 4 + u) ^ (r & 7)) << 4)) = hw4[u];
      }
      stamp(j, 9);
      // coalesced store through a 16-row x 64-byte slab, two passes of 16 rows per warp
#pragma unroll
      for (int ps = 0; ps < 2; ++ps) {
        if ((lane >> 4) == ps) {
          const int sr = lane & 15;  // 16-byte chunks swizzled by (row >> 1) & 3
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(slab + (uint32_t)(sr * 64 + ((u ^ ((sr >> 1) & 3)) << 4))) = hw4[u];
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 2; ++it) {
          const int rr = it * 8 + (lane >> 2), ch = lane & 3;
          const int tok = q * 32 + ps * 16 + rr;
          const uint4 x = *reinterpret_cast<const uint4*>(slab + (uint32_t)(rr * 64 + ((ch ^ ((rr >> 1) & 3)) << 4)));
          if (tok < S)
            st_global_hint(ctx_f16 + (size_t)(row0 + tok) * h + (j0 + j) * 64 + 32 * hf + ch * 8, x, pol_keep);
        }
        __syncwarp();
      }
      stamp(j, 5);
    };
    stamp(0, 6);
    const bool full = S - 64 * hf >= 64;  // warp-uniform
    for (int j = 0; j < hpc; ++j) {  // j: this CTA's head index (absolute head j0 + j)
      if (full)
        softmax(j, std::false_type{});
      else
        softmax(j, std::true_type{});
      epilogue(j);
    }
    // per-token quantize (R1-R3): full-row max-abs from both halves, then
    // warp w re-reads rows 16w..16w+15 (L2), and writes codes + scales
    red[hf * 128 + r] = __half2float(__float2half_rn(amax));
    if (asym) {
      red[256 + hf * 128 + r] = __half2float(__float2half_rn(vmn));
      red[512 + hf * 128 + r] = __half2float(__float2half_rn(vmx));
    }
    __threadfence_block();  // ctx rows written by the other half's warps are re-read below
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (G > 1) goto cluster_tail;  // the row max-abs spans the cluster: combined below
    // The Q/K/V stages are idle now (every MMA completed before the last o_full): warp w
    // stages 6 of its rows at a time (12 KB) with cp.async so ~200 KB per SM is in flight.
    uint8_t* qb = smem + warp * 12288;
    stamp(1, 6);
    for (int r0 = 0; r0 < ((dbg & 1) ? 0 : 16); r0 += 6) {
      const int nr = min(6, 16 - r0);
      for (int rr = 0; rr < nr; ++rr) {
        const int tok = warp * 16 + r0 + rr;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(ctx_f16 + ((size_t)row0 + tok) * h);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (tok < S && lane + 32 * i < h / 8 && !(dbg & 2))
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                             smem_u32(qb + rr * 2048 + (lane + 32 * i) * 16)),
                         "l"(src + (lane + 32 * i) * 16), "l"(pol_drop)
                         : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      if (r0 == 0) stamp(1, 7);
      for (int rr = 0; rr < nr; ++rr) {
        const int tok = warp * 16 + r0 + rr;
        if (tok >= S) continue;
        const float a = fmaxf(red[tok], red[128 + tok]);
        const size_t grow = (size_t)row0 + tok;
        if (asym) {  // O-15 on the fp16 ctx row: zero = min, scale = (max - min) / 15
          const float mn = fminf(red[256 + tok], red[384 + tok]), mx = fmaxf(red[512 + tok], red[640 + tok]);
          uint32_t* cw = reinterpret_cast<uint32_t*>(ctx_codes + grow * (h / 2));
          if (lane == 0) {
            const double D = (double)mx - (double)mn;
            ctx_scales[grow] = D > 0.0 ? (float)(D / 15.0) : 1.0f;
            ctx_zeros[grow] = mn;
          }
          for (int c = lane; c < h / 8; c += 32) {
            const uint4 x = *reinterpret_cast<const uint4*>(qb + rr * 2048 + c * 16);
            const uint32_t hh[4] = {x.x, x.y, x.z, x.w};
            cw[c] = requant8_asym(hh, mn, mx);
          }
          continue;
        }
        if (i8) {  // W8A8 baseline: int8 codes, scale amax/127 (oracle O-11)
          uint2* c8 = reinterpret_cast<uint2*>(ctx_codes + grow * h);
          if (lane == 0) ctx_scales[grow] = a > 0.f ? __fdiv_rn(a, 127.0f) : 1.0f;
          const float rq = a > 0.f ? __fdiv_rn(127.0f, a) : 0.f;
          for (int c = lane; c < h / 8; c += 32) {
            const uint4 x = *reinterpret_cast<const uint4*>(qb + rr * 2048 + c * 16);
            const uint32_t hh[4] = {x.x, x.y, x.z, x.w};
            c8[c] = requant8_i8(hh, a, rq, 0.f);
          }
          continue;
        }
        uint32_t* cw = reinterpret_cast<uint32_t*>(ctx_codes + grow * (h / 2));
        if (lane == 0) ctx_scales[grow] = a > 0.f ? __fdiv_rn(a, 7.0f) : 1.0f;
        if (!(a > 0.f)) {  // all-zero row (R5)
          for (int c = lane; c < h / 8; c += 32) cw[c] = 0u;
          continue;
        }
        const float r7 = __fdiv_rn(7.0f, a);
        // each lane reads back only the chunks it copied; h / 8 = 32 nch chunks per row
        if (dbg & 4) {
          if (!(dbg & 8)) for (int c = lane; c < h / 8; c += 32) cw[c] = 0u;
        } else if (h == 1024) {  // 4 chunks per lane, branch-free fast path
          uint32_t w[4];
          float dmax = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 x = *reinterpret_cast<const uint4*>(qb + rr * 2048 + (lane + 32 * i) * 16);
            const uint32_t hh[4] = {x.x, x.y, x.z, x.w};
            w[i] = requant8_nofix(hh, r7, dmax);
          }
          if (dmax > 0.499998f) {  // near a half-integer somewhere: exact tie-break
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint4 x = *reinterpret_cast<const uint4*>(qb + rr * 2048 + (lane + 32 * i) * 16);
              const uint32_t hh[4] = {x.x, x.y, x.z, x.w};
              w[i] = requant8(hh, a, r7, 0.f);
            }
          }
          if (!(dbg & 8)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) cw[lane + 32 * i] = w[i];
          } else if (w[0] == 0x12345678u && w[1] == 0x9abcdef0u) {
            cw[lane] = w[2] ^ w[3];  // keep the arithmetic live
          }
        } else {
          for (int c = lane; c < h / 8; c += 32) {
            const uint4 x = *reinterpret_cast<const uint4*>(qb + rr * 2048 + c * 16);
            const uint32_t hh[4] = {x.x, x.y, x.z, x.w};
            cw[c] = requant8(hh, a, r7, 0.f);
          }
        }
      }
      if (r0 == 0) stamp(2, 6);
    }
    stamp(0, 7);
  }
cluster_tail:
  if (G > 1) {
    // Row max-abs over the G CTAs of this sequence through distributed shared memory; each
    // CTA then codes its own hpc * 64 columns (a code depends only on its element and the
    // row scale).  All threads of all CTAs take part in both cluster barriers; the second
    // keeps every CTA's red[] alive until the others have read it.
    float* red = reinterpret_cast<float*>(smem + OFF_RED);        // [2][128] this CTA's partials
    float* amx = reinterpret_cast<float*>(smem + OFF_SLAB);       // [128] combined max-abs
    float* rr7 = amx + 128;                                       // [128] 7 / amax
    // One head per CTA, symmetric / int8 codes: PUSH -- each CTA stores its rows' max-abs into
    // slot g of every CTA's gather buffer [G][128] before the cluster barrier (in the second
    // Q/K/V stage, which one head per CTA never loads: a slower peer may still be in its head),
    // so after it every read is local and no CTA touches another's shared memory any more (no
    // second barrier).  Otherwise PULL: remote reads after the barrier, a second barrier
    // before exit.
    const bool push = hpc == 1 && !asym;
    float* gbuf = reinterpret_cast<float*>(smem + STAGE);
    if (push && threadIdx.x < 128) {
      const int r = threadIdx.x;
      const float al = fmaxf(red[r], red[128 + r]);
      const uint32_t la = smem_u32(gbuf + g * 128 + r);
      for (int c = 0; c < G; ++c) st_cluster_f32(mapa(la, (uint32_t)c), al);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    kstamp(2);
    float* zmn = rr7 + 128;                                       // [128] asym: min
    float* zmx = zmn + 128;                                       // [128] asym: max
    if (threadIdx.x < 128) {
      const int r = threadIdx.x;
      float a = 0.f, mn = INFINITY, mx = -INFINITY;
      auto rd = [&](const float* loc, int c) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(loc)), "r"(c));
        float x;
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(ra) : "memory");
        return x;
      };
      if (push) {
        for (int c = 0; c < G; ++c) a = fmaxf(a, gbuf[c * 128 + r]);
      } else if (asym) {
        for (int c = 0; c < G; ++c) {
          a = fmaxf(a, fmaxf(rd(red + r, c), rd(red + 128 + r, c)));
          mn = fminf(mn, fminf(rd(red + 256 + r, c), rd(red + 384 + r, c)));
          mx = fmaxf(mx, fmaxf(rd(red + 512 + r, c), rd(red + 640 + r, c)));
        }
      } else {
        // all 2 G distributed-shared-memory loads in flight before the first use (one round
        // trip instead of 2 G serialised ones; G <= 16)
        float pv[32];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < G) {
            pv[2 * c] = rd(red + r, c);
            pv[2 * c + 1] = rd(red + 128 + r, c);
          }
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < G) a = fmaxf(a, fmaxf(pv[2 * c], pv[2 * c + 1]));
      }
      if (asym) {
        zmn[r] = mn;
        zmx[r] = mx;
        if (g == 0 && r < S) {
          const double D = (double)mx - (double)mn;
          ctx_scales[row0 + r] = D > 0.0 ? (float)(D / 15.0) : 1.0f;
          ctx_zeros[row0 + r] = mn;
        }
      }
      const float qm = i8 ? 127.0f : 7.0f;
      amx[r] = a;
      rr7[r] = a > 0.f ? __fdiv_rn(qm, a) : 0.f;
      if (g == 0 && r < S && !asym) ctx_scales[row0 + r] = a > 0.f ? __fdiv_rn(a, qm) : 1.0f;
    }
    __syncthreads();
    // pull: every remote read of this CTA is done -- arrive now (release), wait only before
    // exit, so the other CTAs' red[] lifetime costs nothing on this CTA's path
    if (!push) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    kstamp(3);
    // this CTA's columns [64 j0, 64 (j0 + hpc)): cpr 16-byte chunks (8 values) per row
    const int cpr = hpc * 8;
    // the ctx chunks this thread codes: the first four loads in flight together (the whole job
    // at one head per CTA: S * 8 chunks over 320 threads), then the rest one by one
    constexpr int PF = 4;
    uint4 xp[PF];
    const bool ctile = hpc == 1;  // the epilogue kept this CTA's ctx tile in shared memory
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int idx = threadIdx.x + u * AT_THREADS;
      if (!ctile && idx < S * cpr) {
        const int rw = idx / cpr, c = idx - rw * cpr;
        xp[u] = __ldcg(reinterpret_cast<const uint4*>(ctx_f16 + (size_t)(row0 + rw) * h + j0 * 64 + c * 8));
      }
    }
    for (int idx = threadIdx.x, u = 0; idx < S * cpr; idx += AT_THREADS, ++u) {
      const int rw = idx / cpr, c = idx - rw * cpr;
      const float a = amx[rw];
      uint4 x;
      if (ctile) {
        x = *reinterpret_cast<const uint4*>(smem + rw * 128 + ((c ^ (rw & 7)) << 4));
      } else if (u < PF) {
#pragma unroll
        for (int k = 0; k < PF; ++k)
          if (k == u) x = xp[k];
      } else {
        x = __ldcg(reinterpret_cast<const uint4*>(ctx_f16 + (size_t)(row0 + rw) * h + j0 * 64 + c * 8));
      }
      const uint32_t hh[4] = {x.x, x.y, x.z, x.w};
      if (asym)
        reinterpret_cast<uint32_t*>(ctx_codes + (size_t)(row0 + rw) * (h / 2) + j0 * 32)[c] = requant8_asym(hh, zmn[rw], zmx[rw]);
      else if (i8)
        reinterpret_cast<uint2*>(ctx_codes + (size_t)(row0 + rw) * h + j0 * 64)[c] = requant8_i8(hh, a, rr7[rw], 0.f);
      else {
        // batched fast requant; near a half-integer the exact per-element tie-break (R2, R3)
        uint32_t wq = 0u;
        if (a > 0.f) {
          float dm = 0.f;
          wq = requant8_nofix(hh, rr7[rw], dm);
          if (dm > 0.499998f) wq = requant8(hh, a, rr7[rw], 0.f);
        }
        reinterpret_cast<uint32_t*>(ctx_codes + (size_t)(row0 + rw) * (h / 2) + j0 * 32)[c] = wq;
      }
    }
    kstamp(4);
    if (!push) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  kstamp(5);
  if (warp == 9) tmem_dealloc(tmem, 256);
}

cudaError_t launch_attention_tc(const __half* qkv, int B, int S, int heads, __half* ctx_f16, uint8_t* ctx_codes,
                                float* ctx_scales, cudaStream_t s, bool i8, float* ctx_zeros) {
  if (B == 0) return cudaSuccess;
  static EncodeFn enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    enc = reinterpret_cast<EncodeFn>(p);
  }
  static bool configured = false;
  if (!configured) {
    for (auto k : {attention_tc_kernel<0>, attention_tc_kernel<1>, attention_tc_kernel<2>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmemMax);
      if (e != cudaSuccess) return e;
      // clusters of up to 16 CTAs (one head per CTA at batch 1); 16 > the portable 8
      e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    configured = true;
  }
  const int h = heads * 64;
  CUtensorMap tq;
  cuuint64_t dims[2] = {(cuuint64_t)(3 * h), (cuuint64_t)B * S};
  cuuint64_t strides[1] = {(cuuint64_t)(3 * h) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(qkv), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static const char* trace_path = prof_env("Q4_TRACE");
  static const int dbg = prof_env("Q4_ATTN_DBG") ? atoi(prof_env("Q4_ATTN_DBG")) : 0;  // profiling only
  static unsigned long long* trace_buf = nullptr;
  if (trace_path && !trace_buf) cudaMalloc(&trace_buf, sizeof(unsigned long long) * 512 * 16 * 16);
  // Small batches: split each sequence's heads over a cluster of G CTAs so the grid fills
  // the GPU (about two CTAs per SM); G divides heads and is at most 8 (portable cluster).
  // Batch <= 4 (the latency configs): up to 16 CTAs per cluster (non-portable), one head per
  // CTA -- BERT-base batch 1, 12 layers: 0.707 -> 0.667 ms eager with G = 12 instead of 6.
  int G = 1;
  if (B < 148)
    for (int d = B <= 4 ? 16 : 8; d >= 2; --d)
      if (heads % d == 0 && B * d <= 296) { G = d; break; }
  static const int g_env = prof_env("Q4_ATTN_G") ? atoi(prof_env("Q4_ATTN_G")) : 0;  // profiling only
  if (g_env > 0 && heads % g_env == 0 && g_env <= 16) G = g_env;
  // profiling only: extra dynamic smem (forces one CTA per SM when SMEM_AT + extra > 114 KB)
  static const int smem_extra = prof_env("Q4_ATTN_SMEM_EXTRA") ? atoi(prof_env("Q4_ATTN_SMEM_EXTRA")) : 0;
  note_launch();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * G));
  cfg.blockDim = dim3(AT_THREADS);
  cfg.dynamicSmemBytes = SMEM_AT + (smem_extra > 0 && SMEM_AT + smem_extra <= kAttnSmemMax ? smem_extra : 0);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see launch_pdl)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = prof_env("Q4_NO_PDL") != nullptr;  // profiling only
  cfg.numAttrs = (no_pdl || (int64_t)B * S > kPdlMaxRows) ? 1 : 2;
  auto kern = ctx_zeros ? attention_tc_kernel<2> : i8 ? attention_tc_kernel<1> : attention_tc_kernel<0>;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, tq, S, heads, ctx_f16, ctx_codes, ctx_scales,
                                      trace_path ? trace_buf : nullptr, dbg, G, ctx_zeros);
  if (le != cudaSuccess && G > 8) {
    // a non-portable cluster the GPU cannot place: fall back to the largest portable one
    (void)cudaGetLastError();
    for (G = 8; G > 1 && heads % G; --G) {}
    cfg.gridDim = dim3((unsigned)(B * G));
    attr[0].val.clusterDim.x = (unsigned)G;
    le = cudaLaunchKernelEx(&cfg, kern, tq, S, heads, ctx_f16, ctx_codes, ctx_scales,
                            trace_path ? trace_buf : nullptr, dbg, G, ctx_zeros);
  }
  if (le != cudaSuccess) return le;
  if (trace_path) {  // profiling only: dump this launch's stamps
    static unsigned long long host[512 * 16 * 16];
    cudaMemcpy(host, trace_buf, sizeof(host), cudaMemcpyDeviceToHost);
    FILE* f = fopen(trace_path, "ab");
    if (f) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
  }
  return cudaGetLastError();
}

}  // namespace q4

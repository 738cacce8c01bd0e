// gemm_tc.cu -- a3..a6: W4A4 linear on the 5th-gen tensor cores (sm_100a).
//
//   acc[m,n] = sum_k qa[m,k] qw[n,k]   exact INT32
//   + fused epilogue: dequant with token x channel scales + bias, then
//     GELU + requant, or residual + LayerNorm + requant.
//
// B200 has no INT4 tensor datapath: INT4 is the HBM/L2 storage format and
// the contraction runs as tcgen05.mma kind::i8.  Persistent, warp-specialized CTA
// (one per SM), 14 warps:
//   warp 0      TMA producer: packed A [128 x 64 B] + B [TN x 64 B] k-blocks -> smem ring
//   warp 1      MMA issuer (one thread): tcgen05.mma kind::i8, M=128, N=TN, K=32, into one
//               of two TMEM accumulators (epilogue of tile i overlaps mainloop of tile i+1)
//   warps 2-5   nibble -> int8 unpack into the UMMA K-major SWIZZLE_128B layout.  K-permutation
//               trick: lo = (w<<4)&0xF0F0F0F0 (even k),
//               hi = w&0xF0F0F0F0 (odd k) -- the same permutation of k for A and B, so the
//               INT32 sum is exactly 256*sum(qa*qw); the 2^-8 folds into the token scale.
//   warps 6-13  epilogue, two groups of 4 warps (column halves of the tile); thread = row
//               (tcgen05.ld 32x32b).  Stores go through a per-warp swizzled smem slab so
//               every global store is a coalesced 128-byte row segment.
// Row epilogues (GELU_Q4 / RESLN_Q4) reduce over the whole output row, which spans
// C = N/TN tiles on C different CTAs: those CTAs process the same m-block at the same
// step and exchange per-row partials (max-abs; shifted LayerNorm moments combined with
// Chan's formula in rank order) through L2 with a per-m-block arrival counter.  The
// grid is sized so all CTAs are co-resident (persistent, <= 1 CTA per SM).
#include <mutex>

#include "kernels.h"

namespace q4 {

enum { EPI_I32 = 0, EPI_F16 = 1, EPI_GELU_Q4 = 2, EPI_RESLN_Q4 = 3 };

struct TcParams {
  int M, N, K;
  int ntn;      // N / TN (tiles along N == CTAs per row group for row epilogues)
  int mblocks;  // ceil(M / 128)
  int groups;   // row epilogues: gridDim.x / ntn
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
  float2* xstat;      // [mblocks][ntn][128] (mean, M2) partials
  float* xamax;       // [mblocks][ntn][128] max-abs partials
  unsigned* xcnt;     // [2][mblocks] arrival counters (zeroed before launch)
};

constexpr int kThreads = 448;
constexpr int kEpiWarp0 = 6;

template <int TN>
struct TcCfg {
  static constexpr int BM = 128, BK = 128;  // BK in int8 elements = 64 packed bytes
  static constexpr int SP = 3, SU = 2;      // packed / unpacked smem stages
  static constexpr int A_PK = BM * 64, B_PK = TN * 64;
  static constexpr int A_UN = BM * 128, B_UN = TN * 128;
  static constexpr int UN_STAGE = A_UN + B_UN, PK_STAGE = A_PK + B_PK;
  static constexpr int OFF_UN = 0;
  static constexpr int OFF_PK = SU * UN_STAGE;
  static constexpr int OFF_STG = OFF_PK + SP * PK_STAGE;  // 8 warps x 4 KB staging slabs
  static constexpr int OFF_ROW = OFF_STG + 8 * 4096;      // [2][128] float4 row partials
  static constexpr int OFF_BAR = OFF_ROW + 2 * 128 * 16;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int HW = TN / 2;  // columns per epilogue group
  static constexpr int TMEM_COLS = 2 * TN <= 64 ? 64 : 2 * TN <= 128 ? 128 : 2 * TN <= 256 ? 256 : 512;
  static_assert(TN % 32 == 0 && TN >= 32 && TN <= 256, "tile N");
  static_assert(SMEM <= 227 * 1024, "smem");
};

// ------------------------------------------------------------------ tile iteration
struct TileIter {
  int cur, step, ntn, mblocks, rank;
  bool row;
  __device__ TileIter(const TcParams& p, bool row_) : ntn(p.ntn), mblocks(p.mblocks), row(row_) {
    if (row) {
      rank = blockIdx.x % p.ntn;
      cur = blockIdx.x / p.ntn;
      step = p.groups;
    } else {
      rank = 0;
      cur = blockIdx.x;
      step = gridDim.x;
    }
  }
  __device__ bool next(int& mb, int& nb) {
    if (row) {
      if (cur >= mblocks) return false;
      mb = cur;
      nb = rank;
    } else {
      if (cur >= mblocks * ntn) return false;
      mb = cur / ntn;
      nb = cur % ntn;
    }
    cur += step;
    return true;
  }
};

// ------------------------------------------------------------------ small helpers
Q4_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
Q4_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
Q4_DEV void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
Q4_DEV void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
// Two INT4 codes -> low byte, previous word shifted left by 8 (I2IP, saturating).
Q4_DEV uint32_t cvt_pack_s4(int hi, int lo, uint32_t prev) {
  uint32_t d;
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(hi), "r"(lo), "r"(prev));
  return d;
}

// Exact symmetric INT4 code of y given the row's (clipped) max-abs a > 0 and r7 = RN(7/a):
// round-half-even of the rational 7y/a (== rint(div.rn(7y, a)), R3).  The fast
// estimate p = y*r7 is within 1e-6 of 7y/a; only when p is that close to a half-integer is
// the side decided exactly by t - a*h with t = 7y, h = the half-integer (exact in fp32 there).
Q4_DEV int requant_code(float y, float a, float r7) {
  const float p = y * r7;
  const float big = 12582912.0f;  // 1.5 * 2^23: (p + big) rounds p to an integer, half-even
  const float s = p + big;
  float fn = s - big;
  int n = __float_as_int(s) - 0x4B400000;
  const float d0 = p - fn;
  if (fabsf(d0) > 0.499998f) {
    const float h = fn + copysignf(0.5f, d0);
    const float e = fmaf(-a, h, 7.0f * y);  // exact: t - a*h
    const int lo = (int)floorf(h), hi = lo + 1;
    n = e > 0.f ? hi : (e < 0.f ? lo : ((lo & 1) ? hi : lo));
  }
  return n;
}

template <int BK>
Q4_DEV void unpack_tile(const uint8_t* __restrict__ pk, uint8_t* __restrict__ un, int rows, int t) {
  constexpr int CPR = BK / 32;  // 16-byte packed chunks per row
  const int n = rows * CPR;
#pragma unroll 4
  for (int i = t; i < n; i += 128) {
    const uint32_t r = (uint32_t)i / CPR, c = (uint32_t)i % CPR;
    const uint4 w = *reinterpret_cast<const uint4*>(pk + (size_t)i * 16);
    uint4 lo, hi;
    lo.x = nib_lo16(w.x); lo.y = nib_lo16(w.y); lo.z = nib_lo16(w.z); lo.w = nib_lo16(w.w);
    hi.x = nib_hi16(w.x); hi.y = nib_hi16(w.y); hi.z = nib_hi16(w.z); hi.w = nib_hi16(w.w);
    uint8_t* row = un + (size_t)r * BK;
    *reinterpret_cast<uint4*>(row + (((2 * c) ^ (r & 7u)) << 4)) = lo;
    *reinterpret_cast<uint4*>(row + (((2 * c + 1) ^ (r & 7u)) << 4)) = hi;
  }
}

// Per-column epilogue parameters for 16 consecutive columns (broadcast loads: every lane
// of the warp reads the same addresses).
Q4_DEV void load_col_params(const float* ws, const __half* bias, float2 (&w)[8], float2 (&b)[8]) {
  const float4* w4 = reinterpret_cast<const float4*>(ws);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 t = __ldg(w4 + j);
    w[2 * j] = make_float2(t.x, t.y);
    w[2 * j + 1] = make_float2(t.z, t.w);
  }
  if (bias) {
    const uint4* b4 = reinterpret_cast<const uint4*>(bias);
    const uint4 u0 = __ldg(b4), u1 = __ldg(b4 + 1);
    const uint32_t u[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = unpack_half2(u[j]);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = make_float2(0.f, 0.f);
  }
}
Q4_DEV void load_half_params(const __half* g, const __half* bt, float2 (&gm)[8], float2 (&be)[8]) {
  const uint4* g4 = reinterpret_cast<const uint4*>(g);
  const uint4* b4 = reinterpret_cast<const uint4*>(bt);
  const uint4 g0 = __ldg(g4), g1 = __ldg(g4 + 1), b0 = __ldg(b4), b1 = __ldg(b4 + 1);
  const uint32_t gu[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  const uint32_t bu[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    gm[j] = unpack_half2(gu[j]);
    be[j] = unpack_half2(bu[j]);
  }
}
// 16 requant codes from 8 packed halves (fast path: FMUL2/FADD2 magic rounding; any value
// within 2e-6 of a half-integer sends the chunk through the exact per-element path).
Q4_DEV void requant16(const uint32_t (&h)[8], float amax, float r7, float clip, int (&qv)[16]) {
  if (!(amax > 0.f)) {
#pragma unroll
    for (int j = 0; j < 16; ++j) qv[j] = 0;
    return;
  }
  float2 y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    y[j] = unpack_half2(h[j]);
    if (clip > 0.f) y[j] = make_float2(fminf(fmaxf(y[j].x, -clip), clip), fminf(fmaxf(y[j].y, -clip), clip));
  }
  const float2 r72 = f2(r7), big = f2(12582912.0f), nbig = f2(-12582912.0f), m1 = f2(-1.0f);
  float dmax = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 pp = fmul2(y[j], r72);
    const float2 sm = fadd2(pp, big);
    const float2 fn = fadd2(sm, nbig);
    const float2 d = ffma2(pp, m1, fn);  // fn - p
    dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
    qv[2 * j] = __float_as_int(sm.x) - 0x4B400000;
    qv[2 * j + 1] = __float_as_int(sm.y) - 0x4B400000;
  }
  if (dmax > 0.499998f) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      qv[2 * j] = requant_code(y[j].x, amax, r7);
      qv[2 * j + 1] = requant_code(y[j].y, amax, r7);
    }
  }
}

// ------------------------------------------------------------------ epilogue pieces
// Per-warp staging slab: 32 rows x 128 bytes, 16-byte chunks XOR-swizzled by row.
Q4_DEV uint32_t slab_off(int row, int chunk) { return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4)); }

// Warp-cooperative coalesced copy of the staged slab (32 rows x `bytes_per_row`, <= 128)
// to global rows [row0, row0+32) at column-byte offset `colb` of a row-major matrix
// with `ldb` bytes per row.
Q4_DEV void slab_store(const uint8_t* stg, uint8_t* gbase, int row0, int M, size_t ldb, size_t colb,
                       int bytes_per_row, int lane) {
  const int cpr = bytes_per_row >> 4;  // 16-byte chunks per row
  const int rows_per_it = 32 / cpr;
  for (int r = lane / cpr; r < 32; r += rows_per_it) {
    const int c = lane % cpr;
    if (row0 + r < M) {
      const uint4 v = *reinterpret_cast<const uint4*>(stg + slab_off(r, c));
      *reinterpret_cast<uint4*>(gbase + (size_t)(row0 + r) * ldb + colb + c * 16) = v;
    }
  }
}
Q4_DEV void slab_load(uint8_t* stg, const uint8_t* gbase, int row0, int M, size_t ldb, size_t colb, int lane) {
  for (int r = lane / 8; r < 32; r += 4) {
    const int c = lane % 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row0 + r < M) v = __ldg(reinterpret_cast<const uint4*>(gbase + (size_t)(row0 + r) * ldb + colb + c * 16));
    *reinterpret_cast<uint4*>(stg + slab_off(r, c)) = v;
  }
}

// Cross-CTA row exchange through L2: publish this CTA's partials, count arrivals of the
// `ntn` CTAs sharing the m-block, wait, then every epilogue thread reads all partials.
Q4_DEV void exchange_sync(unsigned* cnt, int ntn, int ew, int lane) {
  __threadfence();
  named_bar(1, 256);
  if (ew == 0 && lane == 0) {
    atomicAdd(cnt, 1u);
    while (ld_acquire_gpu(cnt) < (unsigned)ntn) __nanosleep(64);
  }
  named_bar(1, 256);
  __threadfence();
}

template <int TN, int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    w4a4_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcParams p) {
  using C = TcCfg<TN>;
  constexpr bool ROW = (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full_p = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty_p = full_p + C::SP;
  uint64_t* full_u = empty_p + C::SP;
  uint64_t* empty_u = full_u + C::SU;
  uint64_t* tfull = empty_u + C::SU;   // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (p.K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::SP; ++i) { mbar_init(&full_p[i], 1); mbar_init(&empty_p[i], 4); }
    for (int i = 0; i < C::SU; ++i) { mbar_init(&full_u[i], 4); mbar_init(&empty_u[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  TileIter it(p, ROW);
  int mb, nb;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      uint32_t g = 0;
      while (it.next(mb, nb)) {
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % C::SP;
          mbar_wait(&empty_p[s], ((g / C::SP) & 1u) ^ 1u);
          uint8_t* pk = smem + C::OFF_PK + s * C::PK_STAGE;
          mbar_arrive_expect_tx(&full_p[s], (uint32_t)C::PK_STAGE);
          tma_load_2d(pk, &tmA, &full_p[s], kb * 64, mb * C::BM);
          tma_load_2d(pk + C::A_PK, &tmB, &full_p[s], kb * 64, nb * TN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_i8(128, TN);
      uint32_t g = 0, tcount = 0;
      while (it.next(mb, nb)) {
        const uint32_t b = tcount & 1u;
        mbar_wait(&tempty[b], ((tcount >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem + b * TN;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int su = g % C::SU;
          mbar_wait(&full_u[su], (g / C::SU) & 1u);
          tc_fence_after();
          const uint32_t ua = smem_u32(smem + C::OFF_UN + su * C::UN_STAGE);
          const uint32_t ub = ua + C::A_UN;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            umma_i8(dt, umma_smem_desc(ua + ks * 32, 1024, 2), umma_smem_desc(ub + ks * 32, 1024, 2), idesc,
                    (kb | ks) != 0);
          umma_commit(&empty_u[su]);
        }
        umma_commit(&tfull[b]);
        ++tcount;
      }
    }
    __syncwarp();
  } else if (warp < kEpiWarp0) {
    // ---------------------------------------------------------------- unpack
    const int t = threadIdx.x - 64;
    uint32_t g = 0;
    while (it.next(mb, nb)) {
      for (int kb = 0; kb < KB; ++kb, ++g) {
        const int s = g % C::SP, su = g % C::SU;
        mbar_wait(&full_p[s], (g / C::SP) & 1u);
        mbar_wait(&empty_u[su], ((g / C::SU) & 1u) ^ 1u);
        const uint8_t* pk = smem + C::OFF_PK + s * C::PK_STAGE;
        uint8_t* un = smem + C::OFF_UN + su * C::UN_STAGE;
        unpack_tile<128>(pk, un, C::BM, t);
        unpack_tile<128>(pk + C::A_PK, un + C::A_UN, TN, t);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full_u[su]);
          mbar_arrive(&empty_p[s]);
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - kEpiWarp0;     // 0..7
    const int grp = ew >> 2;             // column half
    const int q = warp & 3;              // TMEM lane quarter
    const int r = q * 32 + lane;         // row within the tile
    uint8_t* stg = smem + C::OFF_STG + ew * 4096;
    float4* rowp = reinterpret_cast<float4*>(smem + C::OFF_ROW);  // [2][128]
    const int N = p.N;
    const float clip = p.clip;
    uint32_t tcount = 0;
    while (it.next(mb, nb)) {
      const uint32_t b = tcount & 1u;
      const int m0 = mb * C::BM;
      const int gm = m0 + r;
      const bool row_ok = gm < p.M;
      const int c0 = nb * TN + grp * C::HW;  // first global column of this thread's half
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + b * TN + grp * C::HW;
      const float sa = row_ok ? p.a_scales[gm] * (1.0f / 256.0f) : 0.f;
      mbar_wait(&tfull[b], (tcount >> 1) & 1u);
      tc_fence_after();

      if constexpr (KIND == EPI_I32) {
        for (int c = 0; c < C::HW; c += 8) {
          uint32_t v[8];
          tmem_ld8(tbase + c, v);
          tmem_wait_ld();
          if (row_ok) {
            int4* o = reinterpret_cast<int4*>(p.out_i32 + (size_t)gm * N + c0 + c);
            o[0] = make_int4((int)v[0] >> 8, (int)v[1] >> 8, (int)v[2] >> 8, (int)v[3] >> 8);
            o[1] = make_int4((int)v[4] >> 8, (int)v[5] >> 8, (int)v[6] >> 8, (int)v[7] >> 8);
          }
        }
      } else if constexpr (KIND == EPI_F16) {
        const float2 sa2 = f2(sa);
        for (int s0 = 0; s0 < C::HW; s0 += 64) {
          const int sw = C::HW - s0 < 64 ? C::HW - s0 : 64;
          for (int c = 0; c < sw; c += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + s0 + c, v);
            const int n = c0 + s0 + c;
            float2 ws[8], bb[8];
            load_col_params(p.w_scales + n, p.bias ? p.bias + n : nullptr, ws, bb);
            tmem_wait_ld();
            uint32_t h[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float2 t = ffma2(fmul2(make_float2((float)(int)v[2 * j], (float)(int)v[2 * j + 1]), sa2), ws[j], bb[j]);
              h[j] = pack_half2(t.x, t.y);
            }
            *reinterpret_cast<uint4*>(stg + slab_off(lane, c / 8)) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(stg + slab_off(lane, c / 8 + 1)) = make_uint4(h[4], h[5], h[6], h[7]);
          }
          __syncwarp();
          slab_store(stg, reinterpret_cast<uint8_t*>(p.out_f16), m0 + q * 32, p.M, (size_t)N * 2,
                     (size_t)(c0 + s0) * 2, sw * 2, lane);
          __syncwarp();
        }
      } else {
        // ---------------------------------------------------------------- row epilogues
        const int ntn = p.ntn;
        const float2 sa2 = f2(sa);
        float mean = 0.f, rstd = 0.f;
        if constexpr (KIND == EPI_RESLN_Q4) {
          // pass 1: z = acc*sa*sw + b + residual -> TMEM (in place); moments shifted by a pivot
          float2 s1 = f2(0.f), s2 = f2(0.f), npiv = f2(0.f);
          for (int s0 = 0; s0 < C::HW; s0 += 64) {
            const int sw = C::HW - s0 < 64 ? C::HW - s0 : 64;
            slab_load(stg, reinterpret_cast<const uint8_t*>(p.residual), m0 + q * 32, p.M, (size_t)N * 2,
                      (size_t)(c0 + s0) * 2, lane);
            __syncwarp();
            for (int c = 0; c < sw; c += 16) {
              uint32_t v[16];
              tmem_ld16(tbase + s0 + c, v);
              const uint4 ra = *reinterpret_cast<const uint4*>(stg + slab_off(lane, c / 8));
              const uint4 rb = *reinterpret_cast<const uint4*>(stg + slab_off(lane, c / 8 + 1));
              const uint32_t ru[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
              const int n = c0 + s0 + c;
              float2 ws[8], bb[8];
              load_col_params(p.w_scales + n, p.bias ? p.bias + n : nullptr, ws, bb);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float2 t = ffma2(fmul2(make_float2((float)(int)v[2 * j], (float)(int)v[2 * j + 1]), sa2), ws[j], bb[j]);
                const float2 z = fadd2(t, unpack_half2(ru[j]));
                if (s0 == 0 && c == 0 && j == 0) npiv = f2(-z.x);
                const float2 d = fadd2(z, npiv);
                s1 = fadd2(s1, d);
                s2 = ffma2(d, d, s2);
                v[2 * j] = __float_as_uint(z.x);
                v[2 * j + 1] = __float_as_uint(z.y);
              }
              tmem_st16(tbase + s0 + c, v);
            }
            __syncwarp();
          }
          tmem_wait_st();
          // combine the two column halves (Chan), then the ntn CTAs of the row group
          {
            const float nh = (float)C::HW;
            const float S1 = s1.x + s1.y, S2 = s2.x + s2.y;
            const float lmean = -npiv.x + S1 / nh;
            const float lm2 = fmaxf(S2 - S1 * S1 / nh, 0.f);
            rowp[grp * 128 + r] = make_float4(lmean, lm2, 0.f, 0.f);
            named_bar(1, 256);
            const float4 a0 = rowp[r], a1 = rowp[128 + r];
            const float d = a1.x - a0.x;
            const float cm = a0.x + d * 0.5f;
            const float cm2 = a0.y + a1.y + d * d * (nh * 0.5f);
            if (grp == 0) p.xstat[((size_t)mb * ntn + nb) * 128 + r] = make_float2(cm, cm2);
            exchange_sync(p.xcnt + mb, ntn, ew, lane);
            float2 st = __ldcg(&p.xstat[((size_t)mb * ntn) * 128 + r]);
            float cnt = (float)TN;
            mean = st.x;
            float m2 = st.y;
            for (int k = 1; k < ntn; ++k) {
              const float2 o = __ldcg(&p.xstat[((size_t)mb * ntn + k) * 128 + r]);
              const float tot = cnt + (float)TN;
              const float dd = o.x - mean;
              mean = fmaf(dd, (float)TN / tot, mean);
              m2 = m2 + o.y + dd * dd * (cnt * (float)TN / tot);
              cnt = tot;
            }
            rstd = 1.0f / sqrtf(m2 / cnt + p.ln_eps);
          }
        }
        // pass A: y = fp16(GELU(t)) or fp16(LN(z)); row max-abs; y -> TMEM as packed halves
        __half2 hmax = __float2half2_rn(0.f);
        const bool want_f16 = p.out_f16 != nullptr;
        const float2 nmean2 = f2(-mean), rstd2 = f2(rstd);
        for (int s0 = 0; s0 < C::HW; s0 += 64) {
          const int sw = C::HW - s0 < 64 ? C::HW - s0 : 64;
          for (int c = 0; c < sw; c += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + s0 + c, v);
            const int n = c0 + s0 + c;
            uint32_t h[8];
            if constexpr (KIND == EPI_RESLN_Q4) {
              float2 gm[8], bt[8];
              load_half_params(p.gamma + n, p.beta + n, gm, bt);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float2 z = make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
                const float2 y = ffma2(fmul2(fadd2(z, nmean2), rstd2), gm[j], bt[j]);
                h[j] = pack_half2(y.x, y.y);
              }
            } else {
              float2 ws[8], bb[8];
              load_col_params(p.w_scales + n, p.bias ? p.bias + n : nullptr, ws, bb);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float2 t = ffma2(fmul2(make_float2((float)(int)v[2 * j], (float)(int)v[2 * j + 1]), sa2), ws[j], bb[j]);
                const float2 y = gelu2(t);
                h[j] = pack_half2(y.x, y.y);
              }
            }
            if (clip > 0.f) {
              const __half2 cl = __float2half2_rn(clip);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                hmax = __hmax2(hmax, __hmin2(__habs2(*reinterpret_cast<const __half2*>(&h[j])), cl));
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j) hmax = __hmax2(hmax, __habs2(*reinterpret_cast<const __half2*>(&h[j])));
            }
            tmem_st8(tbase + s0 + c, h);
            if (want_f16) {
              *reinterpret_cast<uint4*>(stg + slab_off(lane, c / 8)) = make_uint4(h[0], h[1], h[2], h[3]);
              *reinterpret_cast<uint4*>(stg + slab_off(lane, c / 8 + 1)) = make_uint4(h[4], h[5], h[6], h[7]);
            }
          }
          if (want_f16) {
            __syncwarp();
            slab_store(stg, reinterpret_cast<uint8_t*>(p.out_f16), m0 + q * 32, p.M, (size_t)N * 2,
                       (size_t)(c0 + s0) * 2, sw * 2, lane);
            __syncwarp();
          }
        }
        tmem_wait_st();
        float amax = fmaxf(__low2float(hmax), __high2float(hmax));
        // row max-abs over the two halves and the ntn CTAs
        rowp[grp * 128 + r].z = amax;
        named_bar(1, 256);
        amax = fmaxf(rowp[r].z, rowp[128 + r].z);
        if (grp == 0) p.xamax[((size_t)mb * ntn + nb) * 128 + r] = amax;
        exchange_sync(p.xcnt + p.mblocks + mb, ntn, ew, lane);
        for (int k = 0; k < ntn; ++k) amax = fmaxf(amax, __ldcg(&p.xamax[((size_t)mb * ntn + k) * 128 + r]));
        // pass B: codes (R1-R3), packed, staged, coalesced stores
        const float r7 = amax > 0.f ? __fdiv_rn(7.0f, amax) : 0.f;
        for (int s0 = 0; s0 < C::HW; s0 += 64) {
          const int sw = C::HW - s0 < 64 ? C::HW - s0 : 64;
          for (int c = 0; c < sw; c += 16) {
            uint32_t h[8];
            tmem_ld8(tbase + s0 + c, h);
            tmem_wait_ld();
            int qv[16];
            requant16(h, amax, r7, clip, qv);
            uint32_t w0 = cvt_pack_s4(qv[7], qv[6], 0u);
            w0 = cvt_pack_s4(qv[5], qv[4], w0);
            w0 = cvt_pack_s4(qv[3], qv[2], w0);
            w0 = cvt_pack_s4(qv[1], qv[0], w0);
            uint32_t w1 = cvt_pack_s4(qv[15], qv[14], 0u);
            w1 = cvt_pack_s4(qv[13], qv[12], w1);
            w1 = cvt_pack_s4(qv[11], qv[10], w1);
            w1 = cvt_pack_s4(qv[9], qv[8], w1);
            // 16 codes = 8 bytes; a 64-column slab row holds 32 code bytes in chunks 0-1
            *reinterpret_cast<uint2*>(stg + slab_off(lane, c / 32) + ((c / 16) & 1) * 8) = make_uint2(w0, w1);
          }
          __syncwarp();
          slab_store(stg, p.out_codes, m0 + q * 32, p.M, (size_t)N / 2, (size_t)(c0 + s0) / 2, sw / 2, lane);
          __syncwarp();
        }
        if (row_ok && nb == 0 && grp == 0) p.out_scales[gm] = amax > 0.f ? __fdiv_rn(amax, 7.0f) : 1.0f;
      }
      // accumulator buffer b may be overwritten by the MMA of tile tcount + 2
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      ++tcount;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// ====================================================================== host side

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

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
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t row_bytes, uint32_t box_rows,
               uint32_t box_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int TN, int KIND>
cudaError_t run_tc(const GemmArgs& g, void* ws, size_t ws_bytes, cudaStream_t s, const char** why) {
  using C = TcCfg<TN>;
  auto kern = w4a4_tc_kernel<TN, KIND>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap ta, tb;
  const uint64_t kb = (uint64_t)g.K / 2;
  if (!make_tmap(&ta, g.a_codes, (uint64_t)g.M, kb, 128, 64) || !make_tmap(&tb, g.w_codes, (uint64_t)g.N, kb, TN, 64)) {
    *why = "cuTensorMapEncodeTiled failed (driver entry point or alignment)";
    return cudaErrorInvalidValue;
  }
  TcParams p;
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.ntn = g.N / TN;
  p.mblocks = (g.M + 127) / 128;
  p.a_scales = g.a_scales; p.w_scales = g.w_scales;
  p.bias = g.bias; p.residual = g.residual; p.gamma = g.gamma; p.beta = g.beta;
  p.ln_eps = g.ln_eps; p.clip = g.clip;
  p.out_i32 = g.out_i32; p.out_f16 = g.out_f16; p.out_codes = g.out_codes; p.out_scales = g.out_scales;
  p.xstat = nullptr; p.xamax = nullptr; p.xcnt = nullptr;
  const int sms = num_sms();
  int grid;
  if (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4) {
    // co-residency: one CTA per SM, groups of ntn CTAs; every CTA of a group must be resident
    if (p.ntn > sms) { *why = "row epilogue needs N/TN <= #SMs"; return cudaErrorNotSupported; }
    p.groups = sms / p.ntn;
    if (p.groups > p.mblocks) p.groups = p.mblocks;
    grid = p.groups * p.ntn;
    const size_t need = tc_workspace_bytes(g.M, g.N, TN);
    if (!ws || ws_bytes < need) { *why = "workspace too small for the row-epilogue exchange"; return cudaErrorInvalidValue; }
    uint8_t* w = reinterpret_cast<uint8_t*>(ws);
    const size_t nslot = (size_t)p.mblocks * p.ntn * 128;
    p.xstat = reinterpret_cast<float2*>(w);
    p.xamax = reinterpret_cast<float*>(w + nslot * 8);
    p.xcnt = reinterpret_cast<unsigned*>(w + nslot * 12);
    cudaError_t e = cudaMemsetAsync(p.xcnt, 0, sizeof(unsigned) * 2 * p.mblocks, s);
    if (e != cudaSuccess) return e;
  } else {
    p.groups = 0;
    const int tiles = p.mblocks * p.ntn;
    grid = tiles < sms ? tiles : sms;
  }
  note_launch();
  kern<<<grid, kThreads, C::SMEM, s>>>(ta, tb, p);
  return cudaGetLastError();
}

template <int TN>
cudaError_t run_tc_kind(const GemmArgs& g, void* ws, size_t wsb, cudaStream_t s, const char** why) {
  switch (g.kind) {
    case EPI_I32: return run_tc<TN, EPI_I32>(g, ws, wsb, s, why);
    case EPI_F16: return run_tc<TN, EPI_F16>(g, ws, wsb, s, why);
    case EPI_GELU_Q4: return run_tc<TN, EPI_GELU_Q4>(g, ws, wsb, s, why);
    case EPI_RESLN_Q4: return run_tc<TN, EPI_RESLN_Q4>(g, ws, wsb, s, why);
  }
  *why = "unknown epilogue kind";
  return cudaErrorInvalidValue;
}

}  // namespace

int tc_tile_n(int M, int N, int kind) {
  // Small M (latency configs): narrower tiles spread the work over more SMs.  Row
  // epilogues need >= 64 columns per tile (>= 16 code bytes per row per half).
  const bool row = kind == EPI_GELU_Q4 || kind == EPI_RESLN_Q4;
  const int pref = M <= 512 ? 64 : 256;
  static const int cand[] = {256, 128, 64, 32};
  for (int c : cand)
    if (c <= pref && N % c == 0 && !(row && c < 64)) return c;
  for (int c : cand)
    if (N % c == 0 && !(row && c < 64)) return c;
  return 0;
}

size_t tc_workspace_bytes(int M, int N, int TN) {
  if (TN <= 0) return 0;
  const size_t mblocks = (size_t)(M + 127) / 128, ntn = (size_t)N / TN;
  return mblocks * ntn * 128 * 12 + 2 * mblocks * sizeof(unsigned) + 256;
}

cudaError_t launch_w4a4_tc(const GemmArgs& g, void* ws, size_t ws_bytes, cudaStream_t s, const char** why) {
  if (g.M == 0) return cudaSuccess;
  const int tn = tc_tile_n(g.M, g.N, g.kind);
  if (!tn) {
    *why = "the tcgen05 path needs N % 32 == 0 (N % 64 == 0 for GELU_Q4 / RESLN_Q4)";
    return cudaErrorNotSupported;
  }
  switch (tn) {
    case 256: return run_tc_kind<256>(g, ws, ws_bytes, s, why);
    case 128: return run_tc_kind<128>(g, ws, ws_bytes, s, why);
    case 64: return run_tc_kind<64>(g, ws, ws_bytes, s, why);
    default: return run_tc_kind<32>(g, ws, ws_bytes, s, why);
  }
}

}  // namespace q4

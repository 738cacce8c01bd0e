// gemm_tc.cu -- a3..a6: W4A4 linear on the 5th-gen tensor cores (sm_100a).
//
//   acc[m,n] = sum_k qa[m,k] qw[n,k]   exact INT32
//   + fused epilogue: dequant with token x channel scales + bias, then
//     GELU + requant, or residual + LayerNorm + requant.
//
// B200 has no INT4 tensor datapath: INT4 is the HBM/L2 storage format and
// the contraction runs as tcgen05.mma kind::i8.  Persistent, warp-specialized CTA (one per
// SM); warp roles, in this order so the issue arbiter (which favours higher warp ids)
// prefers the mainloop's critical path:
//   warps 0 .. NE-1   epilogue: two groups of EPW warps (4 for I32 / F16, 8 for the row
//                     epilogues); group g drains TMEM accumulator buffer g, so the epilogue of
//                     tile i overlaps the mainloop of tile i+1; thread = row (tcgen05.ld
//                     32x32b); stores through per-warp swizzled smem slabs (coalesced rows)
//   warps NE .. NE+3  nibble -> int8 unpack into the UMMA K-major SWIZZLE_128B layout.
//                     K-permutation trick: lo = (w<<4)&0xF0F0F0F0
//                     (even k), hi = w&0xF0F0F0F0 (odd k) -- the same permutation of k for A
//                     and B, so the INT32 sum is exactly 256*sum(qa*qw); the 2^-8 folds into
//                     the token scale.  Prepacked weights (BI8) arrive already unpacked.
//   warp NE+4         TMA producer (packed A, B or int8 B stages)
//   warp NE+5         MMA issuer (one thread): tcgen05.mma kind::i8 M=128 (CTA pair: M=256,
//                     cta_group::2, the leader issues for both CTAs), N=TN, K=32, into one of
//                     two TMEM accumulators
// Variants: BI8 (prepacked int8 weights), A8 (W8A8: both operands int8, no unpack), H16
// (fp16 operands, kind::f16: the unquantized parts of a per-part strategy), PAIR (2-CTA
// mainloop for the F16 / I32 epilogues at large M).
// Row epilogues (GELU_Q4 / RESLN_Q4) reduce over the whole output row, which spans
// C = N/TN tiles on C different CTAs: those CTAs process the same m-block at the same
// step and exchange per-row partials (max-abs; shifted LayerNorm moments combined in one
// pass) through L2 with a per-m-block arrival counter.  The grid is sized so all CTAs are
// co-resident (persistent, <= 1 CTA per SM).
// Narrow tiles (TN <= 64, the latency configs, M <= 512): ATM -- the unpack warps write the
// int8 activations straight into TMEM and the MMA reads A from there (TS form); split-K over
// global integer reductions for long k-loops (ksplit); and a single m-block of <= 16 CTAs runs
// as one cluster whose row partials go through distributed shared memory (cx).  DESIGN.md 4.3.
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "../../include/q4.h"
#include "kernels.h"

namespace q4 {

enum { EPI_I32 = 0, EPI_F16 = 1, EPI_GELU_Q4 = 2, EPI_RESLN_Q4 = 3 };
// GELU_Q4 epilogue variant: true = y parked in L2, TMEM released after pass A (gelu_epilogue);
// false = y parked in TMEM, pass B from TMEM after the rendezvous (the shared row-epilogue path)
#ifndef Q4_GELU_DECOUPLED
#define Q4_GELU_DECOUPLED 0
#endif

// split-K only pays for long k-loops (measured, BERT-base batch 1, 12 layers eager: splitting
// the K = 768 GEMMs too costs 0.737 -> 0.727..0.795 ms, the reduction round trip outweighs the
// few k-blocks saved; the K = 3072 FFN2 alone: 0.737 -> 0.707 ms with slices of 4 k-blocks,
// 0.702 with slices of 2): >= kKsplitMinLoop k-blocks of 128, slices of >= kKsplitMinKb
constexpr int kKsplitMaxRows = 256, kKsplitMaxN = 8192, kKsplitMinKb = 2, kKsplitMinLoop = 16;
constexpr size_t kKsplitCntBytes = 1024;  // per m-block: N / TN <= 256 tile counters
int tc_ksplit(int M, int N, int K, int TN, bool row = false);
// CX (single-m-block row GEMMs as one cluster, DSMEM exchange): on; Q4_CX=0 in the profiling
// build disables it (A/B only).
inline bool tc_cx_enabled() {
  static const int env = [] { const char* e = prof_env("Q4_CX"); return e ? atoi(e) : 1; }();
  return env != 0;
}
size_t tc_ksplit_bytes(int M);
size_t tc_counter_bytes(int M);

struct TcParams {
  int M, N, K;
  int ntn;      // N / TN (tiles along N == CTAs per row group for row epilogues)
  int mblocks;  // ceil(M / 128)
  int groups;   // row epilogues: gridDim.x / ntn
  const float* a_scales;
  const float* w_scales;
  const float* a_zeros;  // asymmetric activations (NEXT-3): per-row zero point (min), else nullptr
  const float* w_sums;   // with a_zeros: per-output-channel sum of the weight codes (float, exact)
  const __half* bias;
  const __half* residual;
  const __half* gamma;
  const __half* beta;
  float ln_eps, clip;
  int32_t* out_i32;
  __half* out_f16;
  uint8_t* out_codes;
  float* out_scales;
  float* out_zeros;   // asymmetric requant output (NEXT-3): per-row zero point; nullptr = symmetric
  float2* xmm;        // asymmetric requant: [mblocks][ntn][128] (min, max) partials
  float2* xstat;      // [mblocks][ntn][128] (mean, M2) partials
  float* xamax;       // [mblocks][ntn][128] max-abs partials
  unsigned* xcnt;     // [4][mblocks] arrival / departure counters (self-resetting; zero on entry)
  __half* yscr;       // GELU_Q4 without an fp16 tap: [grid][2 groups][2 slots][128][TN] y parking (L2)
  int pair;           // CTA-pair (cta_group::2) mainloop: cluster of 2, CTA r owns m-block 2 c + r
  int lin;            // linear tile schedule (R4): `groups` units walk the row-major tile order
  int split;          // split-K cluster of two CTAs on the same tiles (SPLIT)
  // split-K over global INT32 reductions (small M, DESIGN.md 4.3 "latency configs"): ksplit CTAs
  // (consecutive blockIdx) share one tile, each runs K / ksplit; each adds its partial into
  // kpart (red.add: integer sums are order-free, so the total is exact) and the last to arrive
  // (kcnt) reads the total back into its TMEM, zeroes kpart / kcnt and runs the unchanged
  // epilogue.  1 = off.
  int ksplit;
  // cluster exchange (CX: one m-block, ntn <= 16 n-tiles, TN <= 64 -- the batch-1 row GEMMs):
  // the ntn CTAs run as one thread-block cluster and push their row partials into every peer's
  // shared memory (st.async, completing on the receiver's mbarrier) instead of the L2 rendezvous
  int cx;
  int32_t* kpart;     // [mblocks][ntn][TN][128] INT32 partial sums (zero at rest)
  unsigned* kcnt;     // [mblocks][ntn] arrivals (zero at rest)
  int dbg;            // profiling only (env Q4_DEBUG_SKIP): 1 skip TMA, 2 skip unpack, 4 skip MMA, 8 skip epilogue math
  unsigned long long* trace;  // profiling only (env Q4_TRACE): [grid][64 tiles][8] %globaltimer stamps
};
Q4_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Epilogue warps per TMEM buffer group: 4 for I32 / F16 (two groups + 6 mainloop warps).
// Row epilogues (GELU_Q4 / RESLN_Q4) run 8 warps per group.  RESLN_Q4 (register-heavy
// LayerNorm passes) rebalances registers with setmaxnreg: the 6 mainloop warps (+2 idle,
// so they form two aligned warpgroups) drop to
// MAINLOOP_REGS and the 16 epilogue warps rise to EPI_REGS.  The pool is what the CTA was
// launched with (768 threads x 80 = 61440): 8 x 48 + 16 x 96 = 1920 warp-registers x 32.
// R4 (row epilogues on the CTA-pair mainloop): four 128-column TMEM accumulators drained by
// four 4-warp groups (thread = row, all 128 columns of the tile), so four tiles are in flight
// per CTA instead of two; the pair MMA (M = 256, N = 128) keeps the shared-memory traffic per
// MAC of the 1-CTA N = 256 tile (each CTA stages half of B).
template <int KIND, bool R4 = false> struct EpiCfg {
  static constexpr bool ROW = KIND == 2 || KIND == 3;
  static constexpr int NBUF = R4 ? 4 : 2;  // TMEM accumulator buffers = epilogue groups
  static constexpr int EPW = R4 ? 4 : ROW ? 8 : 4;
  static constexpr int PAD = (KIND == 3 || (KIND == 2 && (Q4_GELU_DECOUPLED || R4))) ? 2 : 0;  // idle warps completing the mainloop warpgroup
  static constexpr int THREADS = (6 + PAD + NBUF * EPW) * 32;
  static constexpr bool TIGHT = KIND == 2 && Q4_GELU_DECOUPLED && !R4;
  static constexpr int MAINLOOP_REGS = TIGHT ? 56 : 48, EPI_REGS = TIGHT ? 88 : 96;
};

// BI8: B (weights) arrives prepacked as int8 "16*q" in the MMA's K order
// (q4_prepack_weights) and is TMA'd straight into the swizzled operand stage; only the
// activation operand A is unpacked on chip.
// A8 (W8A8 baseline, with BI8): A arrives as int8 codes too and is TMA'd straight into the
// operand stage like B -- no packed ring, no on-chip unpack.
// PAIR (with BI8): CTA-pair mainloop -- tcgen05.mma.cta_group::2 with M = 256; each CTA
// stages its own 128 rows of A and half of the N tile of B, so the B stage halves and the
// unpacked ring deepens to 4 stages.
// SPLIT (small M, narrow tiles): split-K over a cluster of two CTAs; each runs half of the
// k-blocks into its own TMEM accumulator, rank 1 pushes its partial into rank 0's shared memory
// (DSMEM) and rank 0 adds it before the unchanged epilogue -- twice the CTAs for the latency
// configs, whose GEMMs otherwise leave most SMs idle.
template <int TN, bool BI8, bool A8 = false, bool PAIR = false, bool R4 = false, bool SPLIT = false>
struct TcCfg {
  static constexpr int BM = 128, BK = 128;  // BK in int8 elements = 64 packed bytes
  // packed / unpacked smem stages; narrow tiles (the latency configs: few CTAs, each streaming
  // its weight rows from HBM) keep more k-blocks in flight
  // ATM (the narrow small-M tiles with prepacked weights): the unpack warps write the int8
  // activation tile straight into TMEM (tcgen05.st) and the MMA reads A from there (TS form), so
  // A never touches shared memory after its packed TMA stage -- the small-M mainloop is
  // shared-memory bound, and this removes half of its traffic (16 KB written + 16 KB read per
  // k-block).  TMEM: the NBUF accumulators, then SU A stages of 32 columns (128 B of K per row).
  static constexpr bool ATM = BI8 && !A8 && !PAIR && !R4 && !SPLIT && TN <= 64;
  static constexpr int SP = A8 ? 1 : BI8 ? (SPLIT ? 3 : TN <= 64 ? 5 : 4) : 3;
  static constexpr int SU = PAIR ? 4 : ATM ? 4 : BI8 ? (SPLIT ? 3 : TN <= 64 ? 5 : 3) : 2;
  static constexpr int A_PK = A8 ? 0 : BM * 64, B_PK = BI8 ? 0 : TN * 64;
  static constexpr int A_UN = ATM ? 0 : BM * 128, B_UN = (PAIR ? TN / 2 : TN) * 128;
  static constexpr int UN_STAGE = A_UN + B_UN, PK_STAGE = A_PK + B_PK;
  static constexpr int OFF_UN = 0;
  static constexpr int OFF_PK = SU * UN_STAGE;
  static constexpr int NSLAB = R4 ? 16 : 8;              // 4 KB staging slabs: per warp (R4) or warp pair
  static constexpr int OFF_STG = OFF_PK + SP * PK_STAGE;
  static constexpr int OFF_PRM = OFF_STG + NSLAB * 4096;  // [R4 ? 4 groups : 1][5][TN] fp32 column params
  static constexpr int OFF_ROW = OFF_PRM + (R4 ? 4 : 1) * 5 * TN * 4;  // [2 groups][2 sides][128] float4 row partials
  static constexpr int OFF_SRED = OFF_ROW + (R4 ? 0 : 2 * 2 * 128 * 16);  // SPLIT: [2][128][TN] int32 partials
  static constexpr int OFF_CX = OFF_SRED + (SPLIT ? 2 * 128 * TN * 4 : 0);  // CX: [2 exchanges][16][128] float2
  static constexpr int OFF_BAR = OFF_CX + (TN <= 64 && !SPLIT ? 2 * 16 * 128 * 8 : 0);
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
  static constexpr int NBUF = R4 ? 4 : 2;
  static constexpr int ACOL = NBUF * TN;  // ATM: first A-stage column
  static constexpr int TCOLS = NBUF * TN + (ATM ? SU * 32 : 0);
  static constexpr int TMEM_COLS = TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static_assert(TCOLS <= 512, "TMEM");
  static_assert(TN % 32 == 0 && TN >= 32 && TN <= 256, "tile N");
  static_assert(SMEM <= 227 * 1024, "smem");
};

// ------------------------------------------------------------------ tile iteration
struct TileIter {
  // The grid is `groups` x `ntn` CTAs; CTA (g, rank) owns n-block `rank` for the whole
  // kernel and walks m-blocks g, g + groups, ...  (fixed N-tile: column parameters are
  // staged once; row epilogues find the ntn CTAs of an m-block at the same step).
  // CTA pairs: cluster c = blockIdx.x / 2 plays the role of a CTA above over m-block pairs;
  // CTA r of the pair owns m-block 2 * pair + r (M % 256 == 0).
  // Linear schedule (R4): the `groups` units (pairs) take pair-tiles i = unit, unit + groups, ...
  // in row-major (m-block pair, n-block) order, so the ntn tiles of an m-block run in the same
  // or the next wave on consecutive units; every SM is used whatever ntn is.
  int cur, step, mblocks, rank, sub, pair, lin, ntn;
  __device__ TileIter(const TcParams& p) {
    pair = p.pair;
    lin = p.lin;
    ntn = p.ntn;
    const int c = (pair || p.split) ? (int)(blockIdx.x >> 1) : p.ksplit > 1 ? (int)blockIdx.x / p.ksplit : (int)blockIdx.x;
    sub = pair ? (int)(blockIdx.x & 1) : 0;
    mblocks = pair ? p.mblocks / 2 : p.mblocks;
    rank = lin ? 0 : c % p.ntn;
    cur = lin ? c : c / p.ntn;
    step = p.groups;
  }
  __device__ bool next(int& mb, int& nb) {
    if (lin) {
      if (cur >= mblocks * ntn) return false;
      const int mp = cur / ntn;
      nb = cur - mp * ntn;
      mb = pair ? 2 * mp + sub : mp;
      cur += step;
      return true;
    }
    if (cur >= mblocks) return false;
    mb = pair ? 2 * cur + sub : cur;
    nb = rank;
    cur += step;
    return true;
  }
};

// ------------------------------------------------------------------ small helpers
constexpr int kUnpackBar = 12;  // named barrier of the 4 unpack warps (ids 1-11: epilogue)
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
// Unpack `ROWS` rows of one k-block (64 packed bytes -> 128 int8 per row) with 128
// threads.  Chunk i (16 packed bytes = 32 nibbles of row i/4) -> two 16-byte int8 chunks
// (even k, odd k) at swizzled positions.  All loads of a batch are issued before any
// transform/store so each thread keeps NB shared-memory loads in flight.
template <int ROWS>
Q4_DEV void unpack_rows(const uint8_t* __restrict__ pk, uint8_t* __restrict__ un, int t) {
  constexpr int PER = ROWS * 4 / 128;  // 16-byte packed chunks per thread
  static_assert(ROWS * 4 % 128 == 0, "rows");
  // chunk j of thread t: packed row (t >> 2) + 32 j, 16-byte column c = t & 3.  The swizzle
  // key (row & 7) does not depend on j, so both destination offsets are loop-invariant.
  const uint32_t r = (uint32_t)t >> 2, c = (uint32_t)t & 3u, key = r & 7u;
  const uint32_t src = (uint32_t)t * 16;
  const uint32_t d0 = r * 128 + (((2 * c) ^ key) << 4), d1 = r * 128 + (((2 * c + 1) ^ key) << 4);
  constexpr int NB = PER < 8 ? PER : 8;
#pragma unroll
  for (int b0 = 0; b0 < PER; b0 += NB) {
    uint4 w[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) w[j] = *reinterpret_cast<const uint4*>(pk + src + (b0 + j) * 2048);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      uint4 lo, hi;
      lo.x = nib_lo16(w[j].x); lo.y = nib_lo16(w[j].y); lo.z = nib_lo16(w[j].z); lo.w = nib_lo16(w[j].w);
      hi.x = nib_hi16(w[j].x); hi.y = nib_hi16(w[j].y); hi.z = nib_hi16(w[j].z); hi.w = nib_hi16(w[j].w);
      *reinterpret_cast<uint4*>(un + d0 + (b0 + j) * 4096) = lo;
      *reinterpret_cast<uint4*>(un + d1 + (b0 + j) * 4096) = hi;
    }
  }
}

// 32 codes (4 packed words) from 16 words of halves.  Unclipped rows take the batched
// fast path (one tie check per 8 values); clipped rows or near-ties use requant8.
Q4_DEV uint4 requant32(const uint32_t (&h)[16], float amax, float r7, float clip) {
  // The fix-up is taken per 8 codes: a warp holds 32 rows, so a per-32 check sends the whole
  // warp down the exact path for ~20% of its chunks (GELU rows, measured); per 8 it is ~6%.
  uint32_t w[4];
  const bool exact = clip > 0.f || !(amax > 0.f);
  float dm[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t hk[4] = {h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]};
    dm[u] = 0.f;
    w[u] = requant8_nofix(hk, r7, dm[u]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (exact || dm[u] > 0.499998f) {
      const uint32_t hk[4] = {h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]};
      w[u] = requant8(hk, amax, r7, clip);
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
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

// 32 accumulators (raw = 256*acc) of one row -> fp16 of t = acc*sa*sw + b (or GELU(t)),
// packed in 16 words.  Column params come from the group's smem copy (broadcast LDS).
// FACC: the accumulator holds fp32 bits (fp16-operand MMA) instead of an integer.
template <bool FACC = false>
Q4_DEV void dequant32(const uint32_t (&v)[32], float2 sa2, const float* sw, const float* bs, uint32_t (&h)[16],
                      bool gelu = false) {
  const float4* pw = reinterpret_cast<const float4*>(sw);
  const float4* pb = reinterpret_cast<const float4*>(bs);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 w = pw[j], bb = pb[j];
    const float2 a0 = FACC ? make_float2(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]))
                           : make_float2((float)(int)v[4 * j], (float)(int)v[4 * j + 1]);
    const float2 a1 = FACC ? make_float2(__uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]))
                           : make_float2((float)(int)v[4 * j + 2], (float)(int)v[4 * j + 3]);
    float2 t0 = ffma2(fmul2(a0, sa2), make_float2(w.x, w.y), make_float2(bb.x, bb.y));
    float2 t1 = ffma2(fmul2(a1, sa2), make_float2(w.z, w.w), make_float2(bb.z, bb.w));
    if (gelu) {
      t0 = gelu2(t0);
      t1 = gelu2(t1);
    }
    h[2 * j] = pack_half2(t0.x, t0.y);
    h[2 * j + 1] = pack_half2(t1.x, t1.y);
  }
}

// Asymmetric activations (NEXT-3, oracle O-16): t = sw (sa acc + za colsum(qw)) + b.
Q4_DEV void dequant32_asym(const uint32_t (&v)[32], float2 sa2, float2 za2, const float* sw, const float* cs,
                           const float* bs, uint32_t (&h)[16]) {
  const float4* pw = reinterpret_cast<const float4*>(sw);
  const float4* pc = reinterpret_cast<const float4*>(cs);
  const float4* pb = reinterpret_cast<const float4*>(bs);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 w = pw[j], c = pc[j], bb = pb[j];
    const float2 u0 = ffma2(make_float2((float)(int)v[4 * j], (float)(int)v[4 * j + 1]), sa2,
                            fmul2(za2, make_float2(c.x, c.y)));
    const float2 u1 = ffma2(make_float2((float)(int)v[4 * j + 2], (float)(int)v[4 * j + 3]), sa2,
                            fmul2(za2, make_float2(c.z, c.w)));
    const float2 t0 = ffma2(u0, make_float2(w.x, w.y), make_float2(bb.x, bb.y));
    const float2 t1 = ffma2(u1, make_float2(w.z, w.w), make_float2(bb.z, bb.w));
    h[2 * j] = pack_half2(t0.x, t0.y);
    h[2 * j + 1] = pack_half2(t1.x, t1.y);
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

// Cross-CTA row exchange through L2: every thread of the epilogue group has stored its
// partial; one thread publishes the arrival (fence + atomic, cumulative over the group's
// stores via bar.sync), waits for the `ntn` CTAs sharing the m-block, fences again, and
// the group then reads all partials with L2 (.cg) loads.  Same pattern as a grid sync.
// Cross-CTA rendezvous of the ntn CTAs of one m-block (co-resident by construction).
// cnt[0] counts arrivals, cnt[dep] departures; the last CTA to leave resets both, so the
// counters are zero again when the kernel ends (the workspace must be zeroed once before
// its first use; kernels leave it zeroed).  A rendezvous that cannot complete (corrupt
// workspace) traps after ~2^26 polls instead of hanging the GPU.
Q4_DEV void exchange_sync(unsigned* cnt, int ntn, int bar_id, int nthreads, bool leader, int dbg = 0) {
  named_bar(bar_id, nthreads);
  if (leader && !(dbg & 32)) {
    // release-add: the group's partial stores (ordered before it by the bar.sync) become
    // visible with the arrival; the acquire loads order the partial reads after the others'
    // arrivals (same pattern as a grid barrier; no full fences needed)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    unsigned polls = 0;
    while (ld_acquire_gpu(cnt) < (unsigned)ntn) {
      __nanosleep(32);
      if (++polls > (1u << 26)) __trap();
    }
  }
  named_bar(bar_id, nthreads);
}
// Departure from a completed rendezvous (leader only): the last of the ntn CTAs to leave resets
// both counters.  Issued at the end of the tile, off the critical path (12 layers of BERT-base
// at batch 1: 0.663 -> 0.658 ms eager; the large-M row GEMMs 1-2 %): every CTA departs only
// after its own poll saw the full count, and a counter is reused only by the next launch.
Q4_DEV void exchange_depart(unsigned* cnt, size_t dep, int ntn, bool leader, int dbg = 0) {
  if (leader && !(dbg & 32)) {
    if (atomicAdd(cnt + dep, 1u) == (unsigned)ntn - 1) {  // everyone has seen the full count
      cnt[0] = 0u;
      cnt[dep] = 0u;
    }
  }
}
// CX (one m-block as one cluster): push a row partial into slot `dst` of every CTA of the cluster
// (rank c = n-block c), completing on that CTA's mbarrier `bar` (complete_tx, 8 or 4 bytes).
Q4_DEV void cx_push2(const void* dst, float x, float y, const uint64_t* bar, int ntn) {
  const uint32_t la = smem_u32(dst), lb = smem_u32(bar);
  for (int c = 0; c < ntn; ++c)
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
                     mapa(la, (uint32_t)c)),
                 "f"(x), "f"(y), "r"(mapa(lb, (uint32_t)c))
                 : "memory");
}
Q4_DEV void cx_push1(const void* dst, float x, const uint64_t* bar, int ntn) {
  const uint32_t la = smem_u32(dst), lb = smem_u32(bar);
  for (int c = 0; c < ntn; ++c)
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                     mapa(la, (uint32_t)c)),
                 "r"(__float_as_uint(x)), "r"(mapa(lb, (uint32_t)c))
                 : "memory");
}
// CX rendezvous: the leader announces the bytes this CTA receives; one warp of the group waits for
// them; the bar.sync hands the local partials to the whole group
Q4_DEV void cx_wait(uint64_t* bar, uint32_t bytes, bool leader, bool poll_warp, int bar_id, int nthreads) {
  if (leader) mbar_arrive_expect_tx(bar, bytes);
  if (poll_warp) mbar_wait(bar, 0);
  named_bar(bar_id, nthreads);
}

// Partial-slab variant for warps sharing one slab: rows [r0, r0 + nrows).
Q4_DEV void slab_store16(const uint8_t* stg, uint8_t* gbase, int row0, int r0, int nrows, int M, size_t ldb,
                         size_t colb, int bytes_per_row, int lane) {
  const int cpr = bytes_per_row >> 4;
  const int rows_per_it = 32 / cpr;
  for (int r = r0 + lane / cpr; r < r0 + nrows; r += rows_per_it) {
    const int c = lane % cpr;
    if (row0 + r < M) {
      const uint4 v = *reinterpret_cast<const uint4*>(stg + slab_off(r, c));
      *reinterpret_cast<uint4*>(gbase + (size_t)(row0 + r) * ldb + colb + c * 16) = v;
    }
  }
}
Q4_DEV void slab_load16(uint8_t* stg, const uint8_t* gbase, int row0, int r0, int M, size_t ldb, size_t colb,
                        int bytes_per_row, int lane) {
  const int cpr = bytes_per_row >> 4;
  const int rows_per_it = 32 / cpr;
  for (int r = r0 + lane / cpr; r < r0 + 16; r += rows_per_it) {
    const int c = lane % cpr;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row0 + r < M) v = __ldg(reinterpret_cast<const uint4*>(gbase + (size_t)(row0 + r) * ldb + colb + c * 16));
    *reinterpret_cast<uint4*>(stg + slab_off(r, c)) = v;
  }
}

// ------------------------------------------------------------------ GELU_Q4 epilogue
// Decoupled from the accumulator (DESIGN.md 4.3 "GELU_Q4: y parked in L2"):
//   pass A (thread = row, TMEM lane quarter): y = fp16(GELU(acc sa sw + b)) -> global (the
//     fp16 tap if the caller asked for it, else a per-CTA L2 parking slot) through the swizzled
//     slab; per-row partial max-abs.  The TMEM buffer is released right after pass A, so the
//     MMA of tile t + 2 overlaps the rest of tile t's epilogue.
//   publish the partials (red.release) -- no wait here;
//   pass B of the group's PREVIOUS tile t - 2 (warp = 16 rows, lane = 8 columns of a row:
//     coalesced y loads from L2 and coalesced code stores), whose exchange completed while
//     pass A of tile t ran.  The group never idles in the rendezvous.
// Two parking slots per group: y(t) is written before y(t - 2) is consumed.
// Pass B of one tile (m-block pmb, n-block pnb): warp gw of the group codes rows
// [16 gw, 16 gw + 16) of the tile; lane l holds columns [8 l, 8 l + 8) of a row (TN / 8 lanes).
// `ys` is row 0 of the tile's y (ld `ldy` halves), written by this group's pass A.
template <int TN, bool A8, bool H16>
Q4_DEV void gelu_pass_b(const TcParams& p, int pmb, int pnb, const __half* ys, int ldy, int gw, int lane, int gbar,
                        int GT, bool leader) {
  const int ntn = p.ntn;
  if (leader && !(p.dbg & 1024)) {  // rendezvous of m-block pmb (published one group cycle ago)
    unsigned* cnt = p.xcnt + p.mblocks + pmb;
    unsigned polls = 0;
    while (ld_acquire_gpu(cnt) < (unsigned)ntn) {
      __nanosleep(32);
      if (++polls > (1u << 26)) __trap();
    }
    if (atomicAdd(cnt + 2 * (size_t)p.mblocks, 1u) == (unsigned)ntn - 1) {
      cnt[0] = 0u;
      cnt[2 * (size_t)p.mblocks] = 0u;
    }
  }
  named_bar(gbar, GT);
  if (p.dbg & 256) return;
  const int r0 = gw * 16, row0 = pmb * 128 + r0;
  const int nr = p.M - row0 < 16 ? p.M - row0 : 16;  // valid rows of this warp
  const bool act = lane < TN / 8;  // lanes holding columns (all lanes take part in the shuffles)
  // every L2 load of the warp is issued before the first use (one round trip): the 16 y rows
  // (16 B per lane per row), then the ntn max-abs partials of the rows (lanes l and l ^ 16:
  // row l % 16)
  const uint4* yp = reinterpret_cast<const uint4*>(ys + (size_t)r0 * ldy) + lane;
  const int ystep = ldy / 8;
  uint4 y[16];
#pragma unroll
  for (int u = 0; u < 16; ++u)
    if (act && u < nr) y[u] = __ldcg(yp + u * ystep);
  float am = 0.f;
  {
    const float* xp = p.xamax + (size_t)pmb * ntn * 128 + r0 + (lane & 15);
    for (int kk = lane >> 4; kk < ntn; kk += 2) am = fmaxf(am, __ldcg(xp + (size_t)kk * 128));
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 16));
  }
  // lanes 0-15 derive their row's requant multiplier and scale (IEEE divisions) once
  constexpr bool I8 = A8 && !H16;
  constexpr float QMAX = I8 ? 127.0f : 7.0f;
  const float rq_l = am > 0.f ? __fdiv_rn(QMAX, am) : 0.f;
  if (pnb == 0 && lane < nr) p.out_scales[row0 + lane] = am > 0.f ? __fdiv_rn(am, QMAX) : 1.0f;
  // rows whose codes take the exact path (clip, all-zero row)
  const uint32_t exact = __ballot_sync(0xffffffffu, lane < 16 && (p.clip > 0.f || !(am > 0.f)));
  uint8_t* cp = p.out_codes + (size_t)row0 * (I8 ? p.N : p.N / 2) + (I8 ? pnb * TN + 8 * lane : pnb * TN / 2 + 4 * lane);
  const size_t cstep = I8 ? (size_t)p.N : (size_t)p.N / 2;
  const float clip = p.clip;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const float amax = __shfl_sync(0xffffffffu, am, u);
    const float rq = __shfl_sync(0xffffffffu, rq_l, u);
    if (u >= nr) break;
    if (!act) continue;
    const uint32_t hk[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
    if constexpr (I8) {
      *reinterpret_cast<uint2*>(cp + u * cstep) = requant8_i8(hk, amax, rq, clip);
    } else {
      float dm = 0.f;
      uint32_t w = requant8_nofix(hk, rq, dm);
      if (dm > 0.499998f || ((exact >> u) & 1u)) w = requant8(hk, amax, rq, clip);
      *reinterpret_cast<uint32_t*>(cp + u * cstep) = w;
    }
  }
}

// Pass A's y slab (32 rows x 64 fp16, swizzled) -> global: this warp's RS rows from r_first;
// `gq` is row 0 of the slab's 32 rows at the slab's column, `nvalid` the rows < M.
template <int RS>
Q4_DEV void slab_store_y(const uint8_t* stg, uint8_t* gq, int ldb, int r_first, int nvalid, int lane) {
  const int c = lane & 7;
  int r = r_first + (lane >> 3);
  uint8_t* g = gq + r * ldb + c * 16;
#pragma unroll
  for (int i = 0; i < RS / 4; ++i, r += 4, g += 4 * ldb)
    if (r < nvalid) *reinterpret_cast<uint4*>(g) = *reinterpret_cast<const uint4*>(stg + slab_off(r, c));
}

template <int TN, bool A8, bool H16>
Q4_DEV void gelu_epilogue(const TcParams& p, TileIter& it, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                          uint8_t* stg, float4* rowp, const float* prm, int ew, int lane) {
  constexpr int EPW = EpiCfg<EPI_GELU_Q4>::EPW, NS = EPW / 4, GT = EPW * 32;
  constexpr int NSL = TN / 64, RS = 32 / NS;
  const int grp = ew / EPW, sub = (ew >> 2) % NS, q = ew & 3, r = q * 32 + lane;
  const int gw = ew % EPW;  // warp within the group
  const int gbar = 1 + grp, pbar = 4 + grp * 4 + q;
  const bool leader = gw == 0 && lane == 0;
  const float clip = p.clip;
  const bool tap = p.out_f16 != nullptr;
  // y of a tile: the caller's fp16 tap, else this group's two L2 parking slots (alternating)
  const int ldy = tap ? p.N : TN;
  __half* const slot0 = tap ? nullptr : p.yscr + ((size_t)blockIdx.x * 2 + grp) * 2 * 128 * TN;
  auto ybase = [&](int mb, int nb, uint32_t slot) -> __half* {
    return tap ? p.out_f16 + (size_t)mb * 128 * p.N + nb * TN : slot0 + slot * (128 * TN);
  };
  auto slab_sync = [&]() {
    if constexpr (NS > 1) named_bar(pbar, 32 * NS); else __syncwarp();
  };
  // profiling only (Q4_TRACE): per tile [0] acc wait start, [1] acc ready, [2] pass A done (TMEM
  // released), [3] published, [4] pass B start, [6] pass B done
  auto stamp = [&](uint32_t tc, int k) {
    if (p.trace && leader && tc < 64) p.trace[((size_t)blockIdx.x * 64 + tc) * 8 + k] = gtimer();
  };
  uint32_t tcount = 0, slot = 0, ptc = 0;
  int pmb = -1, pnb = 0, mb, nb;
  while (it.next(mb, nb)) {
    const uint32_t b = tcount & 1u;
    if ((int)b != grp) { ++tcount; continue; }
    const int m0 = mb * 128, gm = m0 + r;
    const float sa = gm < p.M ? (H16 ? 1.0f : p.a_scales[gm] * (A8 ? 1.0f : 1.0f / 256.0f)) : 0.f;
    const float2 sa2 = f2(sa);
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + b * TN + 32 * sub;
    uint8_t* yq = reinterpret_cast<uint8_t*>(ybase(mb, nb, slot) + (size_t)(q * 32) * ldy);
    const int qrows = p.M - m0 - q * 32;  // valid rows of this lane quarter (may exceed 32)
    stamp(tcount, 0);
    if (gw == 0) mbar_wait(&tfull[b], (tcount >> 1) & 1u);
    named_bar(gbar, GT);
    tc_fence_after();
    stamp(tcount, 1);
    // pass A: this side's 32-column chunk of each 64-column slab, as two 16-column pieces
    __half2 hmax = __float2half2_rn(0.f);
#pragma unroll 1
    for (int k = 0; k < NSL; ++k) {
#pragma unroll
      for (int hp = 0; hp < 2; ++hp) {
        const int col = 64 * k + 32 * sub + 16 * hp;
        uint32_t v[16], h[8];
        tmem_ld16(tbase + 64 * k + 16 * hp, v);
        tmem_wait_ld_dep(v);
        gelu16<H16>(v, sa2, prm + col, prm + TN + col, h);
        if (clip > 0.f) {
          const __half2 cl = __float2half2_rn(clip);
#pragma unroll
          for (int u = 0; u < 8; ++u) hmax = __hmax2(hmax, __hmin2(__habs2(*reinterpret_cast<const __half2*>(&h[u])), cl));
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) hmax = __hmax2(hmax, __habs2(*reinterpret_cast<const __half2*>(&h[u])));
        }
        const int c16 = 4 * sub + 2 * hp;  // 16-byte chunk of the slab row
        *reinterpret_cast<uint4*>(stg + slab_off(lane, c16)) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(stg + slab_off(lane, c16 + 1)) = make_uint4(h[4], h[5], h[6], h[7]);
      }
      slab_sync();
      if (!(p.dbg & 512)) slab_store_y<RS>(stg, yq + 128 * k, 2 * ldy, RS * sub, qrows, lane);
      slab_sync();
    }
    // the accumulator buffer is free: the MMA of tile tcount + 2 may start
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[b]);
    stamp(tcount, 2);
    float amax = fmaxf(__low2float(hmax), __high2float(hmax));
    if constexpr (NS > 1) {
      rowp[sub * 128 + r].z = amax;
      named_bar(gbar, GT);
      amax = fmaxf(rowp[r].z, rowp[128 + r].z);
    }
    if (sub == 0) p.xamax[((size_t)mb * p.ntn + nb) * 128 + r] = amax;
    // publish: the group's partial stores (ordered by the bar.sync) become visible with the arrival
    named_bar(gbar, GT);
    if (leader) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.xcnt + p.mblocks + mb) : "memory");
    stamp(tcount, 3);
    if (pmb >= 0) {
      stamp(ptc, 4);
      gelu_pass_b<TN, A8, H16>(p, pmb, pnb, ybase(pmb, pnb, slot ^ 1u), ldy, gw, lane, gbar, GT, leader);
      stamp(ptc, 6);
    }
    ptc = tcount;
    pmb = mb;
    pnb = nb;
    slot ^= 1u;
    ++tcount;
  }
  if (pmb >= 0) {
    stamp(ptc, 4);
    gelu_pass_b<TN, A8, H16>(p, pmb, pnb, ybase(pmb, pnb, slot ^ 1u), ldy, gw, lane, gbar, GT, leader);
    stamp(ptc, 6);
  }
}

// H16 (with A8, BI8): fp16 operands (the unquantized parts of a per-part quantization
// strategy).  The byte-level staging is the A8 path unchanged (a 128-byte
// k-block row = 64 fp16), the MMA is kind::f16 with fp32 accumulators, and the epilogue
// reads the accumulator as fp32 with unit scales.
// ASY: a row-epilogue instantiation that also takes asymmetric input (a_zeros) and / or writes
// asymmetric codes (out_zeros), NEXT-3; the symmetric instantiations carry none of that code.
template <int TN, int KIND, bool BI8, bool A8, bool H16 = false, bool PAIR = false, bool ASY = false,
          bool SPLIT = false>
__global__ void __launch_bounds__(EpiCfg<KIND, PAIR && (KIND == 2 || KIND == 3)>::THREADS, 1)
    w4a4_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcParams p) {
  static_assert(!A8 || BI8, "W8A8 takes int8 weights through the BI8 path");
  static_assert(!H16 || A8, "fp16 operands use the A8 staging");
  static_assert(!PAIR || (BI8 && !H16), "pair mainloop: int8 weights");
  // R4: row epilogues on the pair mainloop (four 128-column accumulators, linear schedule)
  constexpr bool R4 = PAIR && (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4);
  static_assert(!R4 || TN == 128, "R4 tiles are 256 x 128 per pair");
  using E = EpiCfg<KIND, R4>;
  static_assert(!(SPLIT && (PAIR || R4)), "split-K runs on the 1-CTA mainloop");
  using C = TcCfg<TN, BI8, A8, PAIR, R4, SPLIT>;
  constexpr int NBUF = E::NBUF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full_p = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty_p = full_p + C::SP;
  uint64_t* full_u = empty_p + C::SP;
  uint64_t* empty_u = full_u + C::SU;
  uint64_t* tfull = empty_u + C::SU;   // [NBUF]
  uint64_t* tempty = tfull + NBUF;     // [NBUF]
  uint64_t* redfull = tempty + NBUF;   // SPLIT [2]: rank 0 -- rank 1's partial of buffer b has landed
  uint64_t* redempty = redfull + 2;    // SPLIT [2]: rank 1 -- rank 0 has consumed it
  uint64_t* cxbar = redempty + 2;      // CX [2]: the ntn partials of exchange 1 / 2 have landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cxbar + 2);
  uint32_t* kflag = tmem_slot + 1;    // [NBUF] split-K: this CTA's slice arrived last

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (p.K + C::BK - 1) / C::BK;
  // CX (cluster exchange) exists only in the narrow 1-CTA instantiations; elsewhere it folds away
  const bool cx = (TN <= 64 && !PAIR && !SPLIT) ? p.cx != 0 : false;
  // Warp roles.  The issue arbiter favours higher warp ids, so the mainloop's critical
  // path (unpack, TMA producer, MMA issuer) sits above the epilogue warps.
  constexpr int NE = NBUF * E::EPW;          // epilogue warps 0 .. NE-1
  constexpr int WU = NE;                     // unpack warps WU .. WU+3
  constexpr int WP = NE + 4;                 // TMA producer
  constexpr int WM = NE + 5;                 // MMA issuer (+ TMEM alloc / dealloc)

  if (warp == WP && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::SP; ++i) { mbar_init(&full_p[i], 1); mbar_init(&empty_p[i], 4); }
    // pair: the leader's full_u counts both CTAs' unpack warps (8) + its producer; its tempty
    // counts both CTAs' epilogue warps
    for (int i = 0; i < C::SU; ++i) { mbar_init(&full_u[i], A8 ? 1 : PAIR ? 9 : BI8 ? 5 : 4); mbar_init(&empty_u[i], 1); }
    for (int i = 0; i < NBUF; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], (PAIR ? 2 : 1) * E::EPW); }
    for (int i = 0; i < 2; ++i) { mbar_init(&redfull[i], E::EPW); mbar_init(&redempty[i], E::EPW); }
    for (int i = 0; i < 2; ++i) mbar_init(&cxbar[i], 1);
    fence_mbar_init();
  }
  if constexpr (PAIR) {
    if (warp == WM) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();  // both CTAs' barriers initialised before any remote arrive
    tc_fence_after();
  } else {
    if (warp == WM) tmem_alloc(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    if (SPLIT || cx) cluster_sync(); else __syncthreads();  // SPLIT / CX: remote arrives need every CTA's barriers
    tc_fence_after();
  }
  const uint32_t crank = (PAIR || SPLIT) ? cluster_ctarank() : 0u;
  // SPLIT: this CTA's half of the k-blocks (rank 0 the first half)
  // split-K over global reductions: slice kslice of p.ksplit (consecutive CTAs share a tile)
  const int ksp = TN <= 64 ? p.ksplit : 1;  // only the narrow small-M tiles split
  const int kslice = ksp > 1 ? (int)(blockIdx.x % (unsigned)ksp) : 0;
  const int kb0 = SPLIT ? (int)crank * (KB / 2) : ksp > 1 ? kslice * KB / ksp : 0;
  const int kb1 = SPLIT ? (crank ? KB : KB / 2) : ksp > 1 ? (kslice + 1) * KB / ksp : KB;
  // pair: shared::cluster address of a barrier in the leader CTA (rank 0)
  auto lead = [&](uint64_t* bar) -> uint32_t { return PAIR ? mapa(smem_u32(bar), 0) : smem_u32(bar); };
  const uint32_t tmem = *tmem_slot;
  TileIter it(p);
  int mb, nb;
  pdl_launch_dependents();
  // everything below may read the previous kernel's outputs -- except the TMA producer's first
  // weight tiles, which it issues before its own wait (the weights are constant)
  if (warp != WP) pdl_wait();

  // Register rebalancing (row epilogues): one setmaxnreg per side, executed by whole
  // warpgroups at a single call site that dominates that side's code.
  if (warp >= NE) {
  if constexpr (E::PAD > 0)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(E::MAINLOOP_REGS));
  if (warp == WP) {
    // ---------------------------------------------------------------- TMA producer
    // Weight (B) tiles of the first k-blocks of the first tile, up to one ring's worth, start
    // before griddepcontrol.wait: under programmatic dependent launch they stream in while the
    // previous kernel is still running (the latency configs' GEMMs wait on their weights).
    uint32_t pre = 0;
    if constexpr (BI8 && !PAIR && !SPLIT) {
      if (lane == 0) {
        TileIter it0(p);
        int mb0, nb0;
        if (it0.next(mb0, nb0))
          for (int kb = kb0; kb < kb1 && pre < (uint32_t)C::SU; ++kb, ++pre) {
            uint8_t* ub = smem + C::OFF_UN + pre * C::UN_STAGE;
            mbar_arrive_expect_tx(&full_u[pre], (uint32_t)(A8 ? C::UN_STAGE : C::B_UN));
            tma_load_2d(ub + C::A_UN, &tmB, &full_u[pre], kb * 128, nb0 * TN);
          }
      }
    }
    pdl_wait();
    if (lane == 0) {
      uint32_t g = 0;
      while (it.next(mb, nb)) {
        if constexpr (A8) {
          // both int8 operands straight into the swizzled MMA stage
          for (int kb = kb0; kb < kb1; ++kb, ++g) {
            const int su = g % C::SU;
            mbar_wait(&empty_u[su], ((g / C::SU) & 1u) ^ 1u);
            uint8_t* ub = smem + C::OFF_UN + su * C::UN_STAGE;
            if constexpr (PAIR) {
              // W8A8 pair: this CTA's A rows and half of the B tile, counted on the leader's barrier
              if (crank == 0) mbar_arrive_expect_tx(&full_u[su], (uint32_t)(2 * C::UN_STAGE));
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(ub)), "l"(reinterpret_cast<uint64_t>(&tmA)),
                  "r"(lead(&full_u[su])), "r"(kb * 128), "r"(mb * C::BM)
                  : "memory");
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(ub + C::A_UN)), "l"(reinterpret_cast<uint64_t>(&tmB)),
                  "r"(lead(&full_u[su])), "r"(kb * 128), "r"(nb * TN + (int)crank * (TN / 2))
                  : "memory");
            } else if (g < pre) {
              tma_load_2d(ub, &tmA, &full_u[su], kb * 128, mb * C::BM);  // B (and the tx count) went first
            } else {
              mbar_arrive_expect_tx(&full_u[su], (uint32_t)C::UN_STAGE);
              tma_load_2d(ub, &tmA, &full_u[su], kb * 128, mb * C::BM);
              tma_load_2d(ub + C::A_UN, &tmB, &full_u[su], kb * 128, nb * TN);
            }
          }
          continue;
        }
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % C::SP;
          mbar_wait(&empty_p[s], ((g / C::SP) & 1u) ^ 1u);
          uint8_t* pk = smem + C::OFF_PK + s * C::PK_STAGE;
          if (p.dbg & 1) {
            mbar_arrive(&full_p[s]);
          } else {
            mbar_arrive_expect_tx(&full_p[s], (uint32_t)C::PK_STAGE);
            tma_load_2d(pk, &tmA, &full_p[s], kb * 64, mb * C::BM);
            if constexpr (!BI8) tma_load_2d(pk + C::A_PK, &tmB, &full_p[s], kb * 64, nb * TN);
          }
          if constexpr (BI8) {
            // int8 weights straight into the (swizzled) operand stage of this k-block
            const int su = g % C::SU;
            if (g < pre) continue;  // issued before griddepcontrol.wait
            mbar_wait(&empty_u[su], ((g / C::SU) & 1u) ^ 1u);
            uint8_t* ub = smem + C::OFF_UN + su * C::UN_STAGE + C::A_UN;
            if constexpr (PAIR) {
              // this CTA's half of the N tile; completion counted on the leader's barrier
              if (crank == 0) mbar_arrive_expect_tx(&full_u[su], (uint32_t)(2 * C::B_UN));
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(ub)), "l"(reinterpret_cast<uint64_t>(&tmB)),
                  "r"(lead(&full_u[su])), "r"(kb * 128), "r"(nb * TN + (int)crank * (TN / 2))
                  : "memory");
            } else {
              mbar_arrive_expect_tx(&full_u[su], (uint32_t)C::B_UN);
              tma_load_2d(ub, &tmB, &full_u[su], kb * 128, nb * TN);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == WM) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && (!PAIR || crank == 0)) {  // pair: the leader issues for both CTAs
      // asymmetric activations: unsigned A codes (a_format bit 7 = 0: u8 x s8)
      const uint32_t idesc = H16 ? umma_idesc_f16kk(128, TN)
                                 : (p.a_zeros ? umma_idesc_i8(PAIR ? 256 : 128, TN) & ~(1u << 7)
                                              : umma_idesc_i8(PAIR ? 256 : 128, TN));
      uint32_t g = 0, tcount = 0;
      // profiling only (Q4_TRACE): per-tile (wait tempty, wait full_u total, issue span), slot 62
      unsigned long long* mtr = p.trace ? p.trace + ((size_t)blockIdx.x * 64 + 62) * 8 : nullptr;
      while (it.next(mb, nb)) {
        const uint32_t b = tcount % NBUF, ph = (tcount / NBUF) & 1u;
        const unsigned long long m0 = mtr ? gtimer() : 0;
        if constexpr (PAIR) mbar_wait_cluster(&tempty[b], ph ^ 1u);
        else mbar_wait(&tempty[b], ph ^ 1u);
        tc_fence_after();
        const unsigned long long m1 = mtr ? gtimer() : 0;
        unsigned long long mw = 0;
        const uint32_t dt = tmem + b * TN;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int su = g % C::SU;
          const unsigned long long w0 = mtr ? gtimer() : 0;
          if constexpr (PAIR) mbar_wait_cluster(&full_u[su], (g / C::SU) & 1u);
          else mbar_wait(&full_u[su], (g / C::SU) & 1u);
          if (mtr) mw += gtimer() - w0;
          tc_fence_after();
          const uint32_t ua = smem_u32(smem + C::OFF_UN + su * C::UN_STAGE);
          const uint32_t ub = ua + C::A_UN;
          if (!(p.dbg & 4)) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              if constexpr (PAIR)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
                    "l"(umma_smem_desc(ua + ks * 32, 1024, 2)), "l"(umma_smem_desc(ub + ks * 32, 1024, 2)),
                    "r"(idesc), "r"((uint32_t)(kb != kb0 || ks != 0))
                    : "memory");
              else if constexpr (H16)
                umma_f16kk(dt, umma_smem_desc(ua + ks * 32, 1024, 2), umma_smem_desc(ub + ks * 32, 1024, 2), idesc,
                           kb != kb0 || ks != 0);
              else if constexpr (C::ATM)  // A from TMEM: 32 k (8 columns) per MMA
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
                    "r"(tmem + C::ACOL + (uint32_t)su * 32 + ks * 8), "l"(umma_smem_desc(ub + ks * 32, 1024, 2)),
                    "r"(idesc), "r"((uint32_t)(kb != kb0 || ks != 0))
                    : "memory");
              else
                umma_i8(dt, umma_smem_desc(ua + ks * 32, 1024, 2), umma_smem_desc(ub + ks * 32, 1024, 2), idesc,
                        kb != kb0 || ks != 0);
            }
          }
          if constexpr (PAIR)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(&empty_u[su])), "h"((uint16_t)3) : "memory");
          else
            umma_commit(&empty_u[su]);
        }
        if constexpr (PAIR)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(smem_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
        else
          umma_commit(&tfull[b]);
        if (mtr && tcount >= 2) {
          const unsigned long long m2 = gtimer();
          mtr[0] += m1 - m0; mtr[1] += mw; mtr[2] += m2 - m1; mtr[3] += 1;
        }
        ++tcount;
      }
    }
    __syncwarp();
  } else if (warp > WM) {
    // idle (register donors completing the mainloop warpgroup)
  } else {
    // ---------------------------------------------------------------- unpack
    const int t = threadIdx.x - 32 * WU;
    uint32_t g = 0;
    // profiling only (Q4_TRACE): k-block phase durations of thread 64, trace slot 63 of this CTA
    unsigned long long* utr = (p.trace && t == 0) ? p.trace + ((size_t)blockIdx.x * 64 + 63) * 8 : nullptr;
    while (!A8 && it.next(mb, nb)) {
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % C::SP, su = g % C::SU;
        const unsigned long long u0 = utr ? gtimer() : 0;
        // Row epilogues: the first unpack warp polls both barriers and the other three block
        // in bar.sync (their spin would take issue slots from 16 busy epilogue warps).  With
        // the light F16 / I32 epilogues every warp polls (measured faster: no barrier hop).
        if (!E::ROW || warp == WU) {
          mbar_wait(&full_p[s], (g / C::SP) & 1u);
          mbar_wait(&empty_u[su], ((g / C::SU) & 1u) ^ 1u);
        }
        const unsigned long long u1 = utr ? gtimer() : 0;
        if constexpr (E::ROW) named_bar(kUnpackBar, 128);
        const unsigned long long u2 = utr ? gtimer() : 0;
        const uint8_t* pk = smem + C::OFF_PK + s * C::PK_STAGE;
        uint8_t* un = smem + C::OFF_UN + su * C::UN_STAGE;
        if constexpr (C::ATM) {
          // row r = this warp's TMEM lane quarter (WU is a multiple of 4); its 64 packed bytes
          // sit in the SWIZZLE_64B TMA stage (16-byte chunk c at c ^ ((r >> 1) & 3): conflict-
          // free) and become 32 TMEM columns in the MMA's K order: per chunk, 16 even-k bytes
          // (lo nibbles, 16 q) then 16 odd-k bytes (hi nibbles) -- the prepacked weights' order
          const int uw = warp - WU, r = 32 * uw + lane;
          const uint8_t* prow = pk + r * 64;
          const uint32_t swz = ((uint32_t)r >> 1) & 3u;
          uint32_t v[32];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 w = *reinterpret_cast<const uint4*>(prow + ((c ^ swz) << 4));
            v[8 * c + 0] = nib_lo16(w.x); v[8 * c + 1] = nib_lo16(w.y);
            v[8 * c + 2] = nib_lo16(w.z); v[8 * c + 3] = nib_lo16(w.w);
            v[8 * c + 4] = nib_hi16(w.x); v[8 * c + 5] = nib_hi16(w.y);
            v[8 * c + 6] = nib_hi16(w.z); v[8 * c + 7] = nib_hi16(w.w);
          }
          tc_fence_after();  // the MMA that read this A stage has completed (empty_u)
          tmem_st32(tmem + ((uint32_t)(32 * uw) << 16) + C::ACOL + su * 32, v);
          tmem_wait_st();
          tc_fence_before();
        } else if (!(p.dbg & 2)) {
          unpack_rows<C::BM>(pk, un, t);
          if constexpr (!BI8) unpack_rows<TN>(pk + C::A_PK, un + C::A_UN, t);
        }
        const unsigned long long u3 = utr ? gtimer() : 0;
        if constexpr (!C::ATM) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR)
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(lead(&full_u[su])) : "memory");
          else
            mbar_arrive(&full_u[su]);
          mbar_arrive(&empty_p[s]);
        }
        if (utr && g >= 16 && g < 16 + 256) {  // (wait_full, wait_empty, unpack, fence+arrive), 256 k-blocks
          const unsigned long long u4 = gtimer();
          utr[0] += u1 - u0; utr[1] += u2 - u1; utr[2] += u3 - u2; utr[3] += u4 - u3; utr[4] += 1;
        }
      }
    }
  }
  } else {
    // ---------------------------------------------------------------- epilogue
    if constexpr (E::PAD > 0)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(E::EPI_REGS));
    // 2 groups (group g drains TMEM buffer g: tiles with tcount % 2 == g) x EPW warps.  In
    // a group, the warp with lane quarter q and side `sub` (EPW = 8: two sides) handles rows
    // 32q..32q+31 and the 32-column chunks j with j % NS == sub.  The NS warps of a
    // (group, q) set share a 32-row x 128-byte staging slab, so every 64-column slab leaves as
    // full 128-byte row segments.
    // R4: 4 groups x 4 warps, group g drains buffer g (tcount % 4 == g); a warp covers its 32
    // rows x all TN = 128 columns and owns a 4 KB slab; column parameters per tile and group.
    constexpr int EPW = E::EPW;
    constexpr int NS = EPW / 4;            // sides per lane quarter
    constexpr int GT = EPW * 32;           // threads per group
    const int ew = warp;                   // 0 .. NBUF*EPW-1
    const int grp = ew / EPW;
    const int sub = (ew >> 2) % NS;
    const int q = warp & 3;                // TMEM lane quarter
    const int r = q * 32 + lane;           // row within the tile
    const int pair = R4 ? ew : grp * 4 + q;  // staging slab
    const int gbar = R4 ? 4 + grp : 1 + grp, pbar = 4 + pair;
    const bool leader = (ew % EPW) == 0 && lane == 0;
    uint8_t* stg = smem + C::OFF_STG + pair * 4096;
    float4* rowp = reinterpret_cast<float4*>(smem + C::OFF_ROW) + grp * 256;  // [2 sides][128]
    const int N = p.N;
    const float clip = p.clip;
    // sw | bias | gamma | beta of this CTA's n-block (staged once) or, R4, of the group's tile
    float* const prm0 = reinterpret_cast<float*>(smem + C::OFF_PRM) + (R4 ? grp * 5 * TN : 0);
    auto load_prm = [&](int c0, int i) {
      prm0[i] = p.w_scales ? p.w_scales[c0 + i] : 1.0f;
      prm0[TN + i] = p.bias ? __half2float(p.bias[c0 + i]) : 0.f;
      if (KIND == EPI_F16 && p.a_zeros) prm0[2 * TN + i] = p.w_sums[c0 + i];
      if (ASY && E::ROW && p.a_zeros) prm0[4 * TN + i] = p.w_sums[c0 + i];  // asymmetric input: colsum
      if constexpr (KIND == EPI_RESLN_Q4) {
        prm0[2 * TN + i] = __half2float(p.gamma[c0 + i]);
        prm0[3 * TN + i] = __half2float(p.beta[c0 + i]);
      }
    };
    if constexpr (!R4) {
      const int c0 = it.rank * TN;  // this CTA's fixed n-block (pairs: per cluster)
      for (int i = ew * 32 + lane; i < TN; i += NBUF * GT) load_prm(c0, i);
      asm volatile("bar.sync 3, %0;" ::"r"(NBUF * GT) : "memory");  // all epilogue warps
    }
    const float* prm = prm0;
    // sync of the NS warps sharing a slab (a warp alone needs only __syncwarp)
    auto slab_sync = [&]() {
      if constexpr (NS > 1) named_bar(pbar, 32 * NS); else __syncwarp();
    };
    constexpr int NCH = TN / 32;          // 32-column chunks per tile
    constexpr int NSL = (NCH + 1) / 2;    // 64-column slabs
    constexpr int RS = 32 / NS;           // slab rows stored by each warp of the set
    uint32_t tcount = 0;
    unsigned long long* tr = nullptr;
    auto stamp = [&](int k) {
      if (tr && leader) tr[k] = gtimer();
    };
    if constexpr (KIND == EPI_GELU_Q4 && Q4_GELU_DECOUPLED && !R4) {
      gelu_epilogue<TN, A8, H16>(p, it, tmem, tfull, tempty, stg, rowp, prm, ew, lane);
    } else
    while (it.next(mb, nb)) {
      const uint32_t b = tcount % NBUF;
      if ((int)b != grp) { ++tcount; continue; }
      tr = (p.trace && tcount < 64) ? p.trace + ((size_t)blockIdx.x * 64 + tcount) * 8 : nullptr;
      if constexpr (R4) load_prm(nb * TN, ew % EPW * 32 + lane);  // GT == TN: one column per thread
      stamp(0);
      const int m0 = mb * C::BM;
      const int gm = m0 + r;
      const bool row_ok = gm < p.M;
      const int c0 = nb * TN;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + b * TN;
      // W4A4: the unpacked operands are 16 q, so the accumulator is 256 x the code sum
      const float sa = row_ok ? (H16 ? 1.0f : p.a_scales[gm] * (A8 ? 1.0f : 1.0f / 256.0f)) : 0.f;
      const float2 sa2 = f2(sa);
      const float2 za2 = f2(row_ok && p.a_zeros ? p.a_zeros[gm] : 0.f);
      const uint4* resp = nullptr;
      uint4 rr[4];  // RESLN: residual of this thread's current chunk (first one loaded before the wait)
      if constexpr (KIND == EPI_RESLN_Q4) {
        // this row's residual chunks: pull them into L2 while the mainloop runs
        resp = reinterpret_cast<const uint4*>(p.residual + (size_t)(row_ok ? gm : 0) * N + c0);
        if (row_ok)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(resp), "r"((uint32_t)TN * 2) : "memory");
#pragma unroll
        for (int u = 0; u < 4; ++u) rr[u] = (row_ok && !(p.dbg & 64)) ? __ldg(resp + 4 * sub + u) : make_uint4(0, 0, 0, 0);
      }
      // one warp of the group polls the accumulator barrier; the others block in bar.sync
      // (a try_wait spin in all EPW warps costs issue slots the working group needs)
      if (ew % EPW == 0) mbar_wait(&tfull[b], (tcount / NBUF) & 1u);
      named_bar(gbar, GT);
      tc_fence_after();
      stamp(1);
      if constexpr (!H16 && !PAIR && TN <= 64) {  // the narrow small-M tiles only
        if (p.ksplit > 1) {
          // split-K over global reductions: add this slice's INT32 partial (coalesced: lane = row),
          // count the arrival; the last slice reads the exact total back into its TMEM.
          const size_t tile = (size_t)mb * p.ntn + nb;
          int32_t* kp = p.kpart + tile * (TN * 128) + r;
          for (int j = sub; j < NCH; j += NS) {
            uint32_t v[32];
            tmem_ld32(tbase + 32 * j, v);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 32; ++u)
              asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(kp + (32 * j + u) * 128), "r"(v[u]) : "memory");
          }
          named_bar(gbar, GT);
          if (leader) {
            unsigned old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.kcnt + tile) : "memory");
            kflag[grp] = old == (unsigned)p.ksplit - 1u;
            if (old == (unsigned)p.ksplit - 1u) p.kcnt[tile] = 0u;  // every slice has arrived: reset
          }
          named_bar(gbar, GT);
          if (!kflag[grp]) {
            // not the last slice: this CTA's part of the tile is done
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
            ++tcount;
            continue;
          }
          for (int j = sub; j < NCH; j += NS) {
            uint32_t v[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = (uint32_t)__ldcg(kp + (32 * j + u) * 128);
#pragma unroll
            for (int u = 0; u < 32; ++u) __stcg(kp + (32 * j + u) * 128, 0);  // zero at rest again
            tmem_st32(tbase + 32 * j, v);
          }
          tmem_wait_st();
        }
      }
      if constexpr (SPLIT) {
        // split-K: sred[b][row] holds rank 1's partial accumulator row, 16-byte chunks XOR-swizzled
        // by row (conflict-free row-per-thread reads); chunks owned as in the epilogue (j = sub + NS i)
        const uint32_t rph = (tcount / NBUF) & 1u;
        uint8_t* srow = smem + C::OFF_SRED + (size_t)b * 128 * TN * 4 + (size_t)r * TN * 4;
        auto soff = [&](int c16) { return (uint32_t)((c16 & ~7) | ((c16 ^ r) & 7)) << 4; };
        if (crank == 1) {
          if (ew % EPW == 0) mbar_wait(&redempty[b], rph ^ 1u);  // rank 0 consumed the previous one
          named_bar(gbar, GT);
          const uint32_t rbase = mapa(smem_u32(srow), 0);
          for (int j = sub; j < TN / 32; j += NS) {
            uint32_t v[32];
            tmem_ld32(tbase + 32 * j, v);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 8; ++u)
              asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + soff(8 * j + u)),
                           "r"(v[4 * u]), "r"(v[4 * u + 1]), "r"(v[4 * u + 2]), "r"(v[4 * u + 3])
                           : "memory");
          }
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&redfull[b]), 0))
                         : "memory");
          // this CTA's accumulator is no longer needed: the MMA of its next tile may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
          ++tcount;
          continue;
        }
        if (ew % EPW == 0) mbar_wait_cluster(&redfull[b], rph);
        named_bar(gbar, GT);
        for (int j = sub; j < TN / 32; j += NS) {
          uint32_t v[32];
          tmem_ld32(tbase + 32 * j, v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 x = *reinterpret_cast<const uint4*>(srow + soff(8 * j + u));
            v[4 * u] += x.x; v[4 * u + 1] += x.y; v[4 * u + 2] += x.z; v[4 * u + 3] += x.w;
          }
          tmem_st32(tbase + 32 * j, v);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&redempty[b]), 1)) : "memory");
        named_bar(gbar, GT);
        tc_fence_after();
      }

      if constexpr (KIND == EPI_I32) {
        for (int j = sub; j < NCH; j += NS) {
          for (int c = 32 * j; c < 32 * j + 32; c += 8) {
            uint32_t v[8];
            tmem_ld8(tbase + c, v);
            tmem_wait_ld();
            if (row_ok) {
              int4* o = reinterpret_cast<int4*>(p.out_i32 + (size_t)gm * N + c0 + c);
              constexpr int SH = A8 ? 0 : 8;
              o[0] = make_int4((int)v[0] >> SH, (int)v[1] >> SH, (int)v[2] >> SH, (int)v[3] >> SH);
              o[1] = make_int4((int)v[4] >> SH, (int)v[5] >> SH, (int)v[6] >> SH, (int)v[7] >> SH);
            }
          }
        }
      } else if constexpr (KIND == EPI_F16) {
        for (int k = 0; k < ((p.dbg & 8) ? 0 : NSL); ++k) {
#pragma unroll
          for (int jj = 0; jj < 2; jj += NS) {
            const int j = 2 * k + jj + sub;
            if (j < NCH) {
              uint32_t v[32];
              tmem_ld32(tbase + 32 * j, v);
              tmem_wait_ld();
              uint32_t h[16];
              if (p.a_zeros)
                dequant32_asym(v, sa2, za2, prm + 32 * j, prm + 2 * TN + 32 * j, prm + TN + 32 * j, h);
              else
                dequant32<H16>(v, sa2, prm + 32 * j, prm + TN + 32 * j, h);
#pragma unroll
              for (int u = 0; u < 4; ++u)
                *reinterpret_cast<uint4*>(stg + slab_off(lane, (j & 1) * 4 + u)) =
                    make_uint4(h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]);
            }
          }
          slab_sync();
          const int cols = TN - 64 * k < 64 ? TN - 64 * k : 64;
          slab_store16(stg, reinterpret_cast<uint8_t*>(p.out_f16), m0 + q * 32, RS * sub, RS, p.M, (size_t)N * 2,
                       (size_t)(c0 + 64 * k) * 2, cols * 2, lane);
          slab_sync();
        }
      } else {
        // ---------------------------------------------------------------- row epilogues
        const int ntn = p.ntn;
        const float inv_ntn = 1.0f / (float)ntn;
        float mean = 0.f, rstd = 0.f;
        if constexpr (KIND == EPI_RESLN_Q4) {
          // pass 1: z = acc*sa*sw + b + residual -> TMEM (in place); moments shifted by a pivot.
          // The residual goes straight to registers, one chunk ahead of its use.
          float2 s1 = f2(0.f), s2 = f2(0.f), npiv = f2(0.f);
          // asymmetric input (O-16: sa acc + za colsum) as a separate instantiation of the
          // loop, so the symmetric path keeps its instruction count
          auto pass1 = [&](auto asym_tag) {
          constexpr bool AS = decltype(asym_tag)::value;
          for (int j = sub; j < NCH; j += NS) {
            uint32_t v[32];
            tmem_ld32(tbase + 32 * j, v);
            uint4 rn[4];
            const bool more = j + NS < NCH;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              rn[u] = (more && row_ok && !(p.dbg & 64)) ? __ldg(resp + 4 * (j + NS) + u) : make_uint4(0, 0, 0, 0);
            const uint32_t ru[16] = {rr[0].x, rr[0].y, rr[0].z, rr[0].w, rr[1].x, rr[1].y, rr[1].z, rr[1].w,
                                     rr[2].x, rr[2].y, rr[2].z, rr[2].w, rr[3].x, rr[3].y, rr[3].z, rr[3].w};
            tmem_wait_ld();
            const float4* pw = reinterpret_cast<const float4*>(prm + 32 * j);
            const float4* pb = reinterpret_cast<const float4*>(prm + TN + 32 * j);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const float4 w = pw[jj], bb = pb[jj];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int e = 4 * jj + 2 * hh;
                const float2 av = H16 ? make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1]))
                                      : make_float2((float)(int)v[e], (float)(int)v[e + 1]);
                float2 sacc;
                if constexpr (AS)
                  sacc = ffma2(av, sa2, fmul2(za2, make_float2(prm[4 * TN + 32 * j + e], prm[4 * TN + 32 * j + e + 1])));
                else
                  sacc = fmul2(av, sa2);
                const float2 t = ffma2(sacc, hh ? make_float2(w.z, w.w) : make_float2(w.x, w.y),
                                       hh ? make_float2(bb.z, bb.w) : make_float2(bb.x, bb.y));
                const float2 z = add_half2_f32(ru[e / 2], t);
                if (j == sub && e == 0) npiv = f2(-z.x);
                const float2 d = fadd2(z, npiv);
                s1 = fadd2(s1, d);
                s2 = ffma2(d, d, s2);
                v[e] = __float_as_uint(z.x);
                v[e + 1] = __float_as_uint(z.y);
              }
            }
            tmem_st32(tbase + 32 * j, v);
#pragma unroll
            for (int u = 0; u < 4; ++u) rr[u] = rn[u];
          }
          };
          if (ASY && p.a_zeros) pass1(std::true_type{}); else pass1(std::false_type{});
          tmem_wait_st();
          stamp(2);
          {
            // this side's (mean, M2); combine the sides (Chan), then the ntn CTAs (Chan, rank order)
            const float nh = (float)(TN / NS);
            const float S1 = s1.x + s1.y, S2 = s2.x + s2.y;
            float cm = -npiv.x + S1 / nh, cm2 = fmaxf(S2 - S1 * S1 / nh, 0.f);
            if constexpr (NS > 1) {
              rowp[sub * 128 + r] = make_float4(cm, cm2, 0.f, 0.f);
              named_bar(gbar, GT);
              const float4 a0 = rowp[r], a1 = rowp[128 + r];
              const float d = a1.x - a0.x;
              cm = a0.x + 0.5f * d;
              cm2 = a0.y + a1.y + d * d * (nh * 0.5f);
            }
            float2* gx1 = reinterpret_cast<float2*>(smem + C::OFF_CX);  // CX: [16][128]
            if (cx) {
              if (sub == 0) cx_push2(gx1 + nb * 128 + r, cm, cm2, &cxbar[0], ntn);
              cx_wait(&cxbar[0], (uint32_t)ntn * 128 * 8, leader, ew % EPW == 0, gbar, GT);
            } else {
              if (sub == 0) p.xstat[((size_t)mb * ntn + nb) * 128 + r] = make_float2(cm, cm2);
              exchange_sync(p.xcnt + mb, ntn, gbar, GT, leader, p.dbg);
            }
            stamp(3);
            // every partial covers TN columns: mean = average of the means, M2 = sum of the M2s
            // + TN * sum of squared deviations of the means.  One pass, deviations taken
            // from partial 0's mean (the partial means are close, so no cancellation).
            const float2* xs = p.xstat + ((size_t)mb * ntn) * 128 + r;
            const float2* xl = gx1 + r;
            const float2 o0 = cx ? xl[0] : __ldcg(xs);
            float dsum = 0.f, dsq = 0.f, m2 = o0.y;
            for (int kk = 1; kk < ntn; ++kk) {
              const float2 o = cx ? xl[kk * 128] : __ldcg(xs + (size_t)kk * 128);
              const float dd = o.x - o0.x;
              dsum += dd;
              dsq = fmaf(dd, dd, dsq);
              m2 += o.y;
            }
            const float dm = dsum * inv_ntn;  // mean - mean_0
            mean = o0.x + dm;
            m2 = fmaf((float)TN, fmaf(-(float)ntn * dm, dm, dsq), m2);
            const float cnt = (float)(TN * ntn);
            rstd = 1.0f / sqrtf(m2 / cnt + p.ln_eps);
          }
        }
        // pass A: y = fp16(GELU(t)) or fp16(LN(z)); row max-abs; y -> TMEM as packed halves
        __half2 hmax = __float2half2_rn(0.f);
        // asymmetric output (NEXT-3): the row min and max of y instead of max |y|
        const bool aout = ASY && !A8 && p.out_zeros != nullptr;
        __half2 hmn = __float2half2_rn(65504.f), hmx = __float2half2_rn(-65504.f);
        const bool want_f16 = p.out_f16 != nullptr;
        const float2 nmean2 = f2(-mean), rstd2 = f2(rstd);
        for (int k = 0; k < NSL; ++k) {
#pragma unroll
          for (int jj = 0; jj < 2; jj += NS) {
            const int j = 2 * k + jj + sub;
            uint32_t v[32];
            tmem_ld32(tbase + 32 * j, v);
            tmem_wait_ld();
            uint32_t h[16];
            if constexpr (KIND == EPI_RESLN_Q4) {
              const float4* pg = reinterpret_cast<const float4*>(prm + 2 * TN + 32 * j);
              const float4* pe = reinterpret_cast<const float4*>(prm + 3 * TN + 32 * j);
#pragma unroll
              for (int i4 = 0; i4 < 8; ++i4) {
                const float4 g4 = pg[i4], e4 = pe[i4];
                const float2 z0 = make_float2(__uint_as_float(v[4 * i4]), __uint_as_float(v[4 * i4 + 1]));
                const float2 z1 = make_float2(__uint_as_float(v[4 * i4 + 2]), __uint_as_float(v[4 * i4 + 3]));
                const float2 y0 = ffma2(fmul2(fadd2(z0, nmean2), rstd2), make_float2(g4.x, g4.y), make_float2(e4.x, e4.y));
                const float2 y1 = ffma2(fmul2(fadd2(z1, nmean2), rstd2), make_float2(g4.z, g4.w), make_float2(e4.z, e4.w));
                h[2 * i4] = pack_half2(y0.x, y0.y);
                h[2 * i4 + 1] = pack_half2(y1.x, y1.y);
              }
            } else {
              uint32_t v0[16], v1[16], h0[8], h1[8];
#pragma unroll
              for (int u = 0; u < 16; ++u) { v0[u] = v[u]; v1[u] = v[16 + u]; }
              if (ASY && p.a_zeros) {  // asymmetric input (O-16)
                gelu16<H16, true>(v0, sa2, prm + 32 * j, prm + TN + 32 * j, h0, za2, prm + 4 * TN + 32 * j);
                gelu16<H16, true>(v1, sa2, prm + 32 * j + 16, prm + TN + 32 * j + 16, h1, za2, prm + 4 * TN + 32 * j + 16);
              } else {
                gelu16<H16>(v0, sa2, prm + 32 * j, prm + TN + 32 * j, h0);
                gelu16<H16>(v1, sa2, prm + 32 * j + 16, prm + TN + 32 * j + 16, h1);
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) { h[u] = h0[u]; h[8 + u] = h1[u]; }
            }
            if (aout) {
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                hmn = __hmin2(hmn, *reinterpret_cast<const __half2*>(&h[u]));
                hmx = __hmax2(hmx, *reinterpret_cast<const __half2*>(&h[u]));
              }
            } else if (clip > 0.f) {
              const __half2 cl = __float2half2_rn(clip);
#pragma unroll
              for (int u = 0; u < 16; ++u)
                hmax = __hmax2(hmax, __hmin2(__habs2(*reinterpret_cast<const __half2*>(&h[u])), cl));
            } else {
#pragma unroll
              for (int u = 0; u < 16; ++u) hmax = __hmax2(hmax, __habs2(*reinterpret_cast<const __half2*>(&h[u])));
            }
            tmem_st16(tbase + 32 * j, h);
            if (want_f16) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                *reinterpret_cast<uint4*>(stg + slab_off(lane, (j & 1) * 4 + u)) =
                    make_uint4(h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]);
            }
          }
          if (want_f16) {
            slab_sync();
            slab_store16(stg, reinterpret_cast<uint8_t*>(p.out_f16), m0 + q * 32, RS * sub, RS, p.M, (size_t)N * 2,
                         (size_t)(c0 + 64 * k) * 2, 128, lane);
            slab_sync();
          }
        }
        tmem_wait_st();
        stamp(4);
        if (aout) {
          // asymmetric requant (O-15 on the fp16 row): row (min, max) over the sides, then the ntn
          // CTAs; codes = rhe(15 (y - min) / (max - min)) with the exact fp64 tie-break
          float mn = fminf(__low2float(hmn), __high2float(hmn)), mx = fmaxf(__low2float(hmx), __high2float(hmx));
          if constexpr (NS > 1) {
            rowp[sub * 128 + r].z = mn;
            rowp[sub * 128 + r].w = mx;
            named_bar(gbar, GT);
            mn = fminf(rowp[r].z, rowp[128 + r].z);
            mx = fmaxf(rowp[r].w, rowp[128 + r].w);
          }
          float2* gx2 = reinterpret_cast<float2*>(smem + C::OFF_CX + 16 * 128 * 8);  // CX: [16][128]
          if (cx) {
            if (sub == 0) cx_push2(gx2 + nb * 128 + r, mn, mx, &cxbar[1], ntn);
            cx_wait(&cxbar[1], (uint32_t)ntn * 128 * 8, leader, ew % EPW == 0, gbar, GT);
          } else {
            if (sub == 0) p.xmm[((size_t)mb * ntn + nb) * 128 + r] = make_float2(mn, mx);
            exchange_sync(p.xcnt + p.mblocks + mb, ntn, gbar, GT, leader, p.dbg);
          }
          for (int kk = 0; kk < ntn; ++kk) {
            const float2 o = cx ? gx2[kk * 128 + r] : __ldcg(&p.xmm[((size_t)mb * ntn + kk) * 128 + r]);
            mn = fminf(mn, o.x);
            mx = fmaxf(mx, o.y);
          }
          for (int j = sub; j < NCH; j += NS) {
            uint32_t h[16];
            tmem_ld16(tbase + 32 * j, h);
            tmem_wait_ld();
            uint32_t w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t hk[4] = {h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]};
              w[u] = requant8_asym(hk, mn, mx);
            }
            *reinterpret_cast<uint4*>(stg + slab_off(lane, j)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
          slab_sync();
          slab_store16(stg, p.out_codes, m0 + q * 32, RS * sub, RS, p.M, (size_t)N / 2, (size_t)c0 / 2, TN / 2, lane);
          slab_sync();
          if (row_ok && nb == 0 && sub == 0) {
            const double D = (double)mx - (double)mn;
            p.out_scales[gm] = D > 0.0 ? (float)(D / 15.0) : 1.0f;
            p.out_zeros[gm] = mn;
          }
        } else {
        float amax = fmaxf(__low2float(hmax), __high2float(hmax));
        // row max-abs over the sides, then the ntn CTAs
        if constexpr (NS > 1) {
          rowp[sub * 128 + r].z = amax;
          named_bar(gbar, GT);
          amax = fmaxf(rowp[r].z, rowp[128 + r].z);
        }
        float* gxa = reinterpret_cast<float*>(smem + C::OFF_CX + 16 * 128 * 8);  // CX: [16][128]
        if (cx) {
          if (sub == 0) cx_push1(gxa + nb * 128 + r, amax, &cxbar[1], ntn);
          cx_wait(&cxbar[1], (uint32_t)ntn * 128 * 4, leader, ew % EPW == 0, gbar, GT);
          for (int kk = 0; kk < ntn; ++kk) amax = fmaxf(amax, gxa[kk * 128 + r]);
        } else {
          if (sub == 0) p.xamax[((size_t)mb * ntn + nb) * 128 + r] = amax;
          exchange_sync(p.xcnt + p.mblocks + mb, ntn, gbar, GT, leader, p.dbg);
          // narrow tiles (batch 1: up to 48 partials) keep every load in flight at once
#pragma unroll(TN <= 64 ? 48 : 16)
          for (int kk = 0; kk < ntn; ++kk) amax = fmaxf(amax, __ldcg(&p.xamax[((size_t)mb * ntn + kk) * 128 + r]));
        }
        stamp(5);
        // pass B: codes (R1-R3), packed, staged, coalesced stores
        if constexpr (A8 && !H16) {
          // W8A8: int8 codes (O-11), 64 bytes per 64-column slab row
          const float rq = amax > 0.f ? __fdiv_rn(127.0f, amax) : 0.f;
          for (int k = 0; k < NSL; ++k) {
#pragma unroll
            for (int jj = 0; jj < 2; jj += NS) {
              const int j = 2 * k + jj + sub;
              uint32_t h[16];
              tmem_ld16(tbase + 32 * j, h);
              tmem_wait_ld();
              uint2 c8[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint32_t hk[4] = {h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]};
                c8[u] = requant8_i8(hk, amax, rq, clip);
              }
              *reinterpret_cast<uint4*>(stg + slab_off(lane, 2 * (j & 1))) = make_uint4(c8[0].x, c8[0].y, c8[1].x, c8[1].y);
              *reinterpret_cast<uint4*>(stg + slab_off(lane, 2 * (j & 1) + 1)) = make_uint4(c8[2].x, c8[2].y, c8[3].x, c8[3].y);
            }
            slab_sync();
            slab_store16(stg, p.out_codes, m0 + q * 32, RS * sub, RS, p.M, (size_t)N, (size_t)(c0 + 64 * k), 64, lane);
            slab_sync();
          }
          if (row_ok && nb == 0 && sub == 0) p.out_scales[gm] = amax > 0.f ? __fdiv_rn(amax, 127.0f) : 1.0f;
        } else {
        const float r7 = amax > 0.f ? __fdiv_rn(7.0f, amax) : 0.f;
        // the whole tile row's codes (TN / 2 <= 128 bytes) fit one slab row: chunk j -> slab
        // chunk j, then one synchronised store of full row segments
        for (int j = sub; j < NCH; j += NS) {
          uint32_t h[16];
          tmem_ld16(tbase + 32 * j, h);
          tmem_wait_ld();
          *reinterpret_cast<uint4*>(stg + slab_off(lane, j)) = requant32(h, amax, r7, clip);
        }
        slab_sync();
        slab_store16(stg, p.out_codes, m0 + q * 32, RS * sub, RS, p.M, (size_t)N / 2, (size_t)c0 / 2, TN / 2, lane);
        slab_sync();
        if (row_ok && nb == 0 && sub == 0) p.out_scales[gm] = amax > 0.f ? __fdiv_rn(amax, 7.0f) : 1.0f;
        }
        }
      }
      if (E::ROW && !cx) {
        // leave this m-block's rendezvous (off the critical path: after every partial read)
        if constexpr (KIND == EPI_RESLN_Q4) exchange_depart(p.xcnt + mb, 2 * (size_t)p.mblocks, p.ntn, leader, p.dbg);
        exchange_depart(p.xcnt + p.mblocks + mb, 2 * (size_t)p.mblocks, p.ntn, leader, p.dbg);
      }
      stamp(6);
      // accumulator buffer b may be overwritten by the MMA of tile tcount + 2
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(lead(&tempty[b])) : "memory");
        else
          mbar_arrive(&tempty[b]);
      }
      ++tcount;
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) {
    cluster_sync();  // the leader's MMAs write this CTA's TMEM and read its smem until the end
    if (warp == WM)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
  } else {
    if constexpr (SPLIT) cluster_sync();  // rank 1's remote stores / arrives into rank 0 have landed
    if (warp == WM) tmem_dealloc(tmem, C::TMEM_COLS);
  }
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
               uint32_t box_bytes, bool swizzle128 = false, bool swizzle64 = false) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : swizzle64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

template <int TN, int KIND, bool BI8, bool A8, bool H16 = false, bool PAIR = false, bool ASY = false,
          bool SPLIT = false>
cudaError_t run_tc(const GemmArgs& g, void* ws, size_t ws_bytes, cudaStream_t s, const char** why) {
  constexpr bool R4 = PAIR && (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4);
  using C = TcCfg<TN, BI8, A8, PAIR, R4, SPLIT>;
  constexpr int THREADS = EpiCfg<KIND, R4>::THREADS;
  auto kern = w4a4_tc_kernel<TN, KIND, BI8, A8, H16, PAIR, ASY, SPLIT>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    if constexpr (!PAIR && !SPLIT && TN <= 64) {  // CX clusters of up to 16 CTAs (> the portable 8)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    configured = true;
  }
  CUtensorMap ta, tb;
  const uint64_t kb = (uint64_t)g.K / 2;
  const bool okb = BI8 ? make_tmap(&tb, g.w_i8, (uint64_t)g.N, (uint64_t)g.K, PAIR ? TN / 2 : TN, 128, true)
                       : make_tmap(&tb, g.w_codes, (uint64_t)g.N, kb, TN, 64);
  const bool oka = A8 ? make_tmap(&ta, g.a_i8, (uint64_t)g.M, (uint64_t)g.K, 128, 128, true)
                     : make_tmap(&ta, g.a_codes, (uint64_t)g.M, kb, 128, 64, false, C::ATM);
  if (!oka || !okb) {
    *why = "cuTensorMapEncodeTiled failed (driver entry point or alignment)";
    return cudaErrorInvalidValue;
  }
  TcParams p;
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.ntn = g.N / TN;
  p.mblocks = (g.M + 127) / 128;
  p.a_scales = g.a_scales; p.w_scales = g.w_scales;
  p.a_zeros = g.a_zeros; p.w_sums = g.w_sums;
  p.pair = PAIR ? 1 : 0;
  p.lin = R4 ? 1 : 0;
  p.split = SPLIT ? 1 : 0;
  p.ksplit = 1; p.kpart = nullptr; p.kcnt = nullptr; p.cx = 0;
  p.bias = g.bias; p.residual = g.residual; p.gamma = g.gamma; p.beta = g.beta;
  p.ln_eps = g.ln_eps; p.clip = g.clip;
  p.out_i32 = g.out_i32; p.out_f16 = g.out_f16; p.out_codes = g.out_codes; p.out_scales = g.out_scales;
  p.out_zeros = g.out_zeros;
  p.xstat = nullptr; p.xamax = nullptr; p.xcnt = nullptr; p.yscr = nullptr; p.xmm = nullptr;
  static const int dbg = [] { const char* e = prof_env("Q4_DEBUG_SKIP"); return e ? atoi(e) : 0; }();
  p.dbg = dbg;
  p.trace = nullptr;
  static const char* trace_path = prof_env("Q4_TRACE");
  static unsigned long long* trace_buf = nullptr;
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, sizeof(unsigned long long) * 148 * 64 * 8);
    cudaMemsetAsync(trace_buf, 0, sizeof(unsigned long long) * 148 * 64 * 8, s);
    p.trace = trace_buf;
  }
  const int sms = num_sms();
  // groups of ntn co-resident CTAs (one per SM); a group walks the m-blocks.  Pairs: the unit
  // is a 2-CTA cluster (two SMs) walking m-block pairs.
  const int units = (PAIR || SPLIT) ? sms / 2 : sms, mwalk = PAIR ? p.mblocks / 2 : p.mblocks;
  int grid;
  if constexpr (R4) {
    // linear schedule over every co-resident CTA pair (the row rendezvous spins, so all
    // clusters must be resident at once: the occupancy query bounds the grid)
    static const int max_clusters = [&] {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * units);
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = C::SMEM;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = 0;
      return n;
    }();
    if (max_clusters <= 0) { *why = "no co-resident CTA pair for the R4 kernel"; return cudaErrorNotSupported; }
    p.groups = max_clusters < units ? max_clusters : units;
    if (p.groups > mwalk * p.ntn) p.groups = mwalk * p.ntn;
    grid = 2 * p.groups;
  } else {
    if (p.ntn > units) { *why = "N/TN exceeds the number of SMs"; return cudaErrorNotSupported; }
    if constexpr (!PAIR && !SPLIT && !H16 && TN <= 64) {
      // split-K over global reductions (small M): needs the workspace's zero-at-rest prefix
      const int ks = tc_ksplit(g.M, g.N, g.K, TN, KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4);
      const size_t cb = tc_counter_bytes(g.M);
      if (ks > 1 && ws && ws_bytes >= cb + tc_ksplit_bytes(g.M)) {
        uint8_t* w = reinterpret_cast<uint8_t*>(ws) + cb;
        p.ksplit = ks;
        p.kcnt = reinterpret_cast<unsigned*>(w);
        p.kpart = reinterpret_cast<int32_t*>(w + (size_t)p.mblocks * kKsplitCntBytes);
      }
    }
    p.groups = units / (p.ntn * p.ksplit);
    if (p.groups > mwalk) p.groups = mwalk;
    grid = p.groups * p.ntn * p.ksplit * ((PAIR || SPLIT) ? 2 : 1);
  }
  if (KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4) {
    const size_t need = tc_workspace_bytes(g.M, g.N, TN, KIND);
    if (!ws || ws_bytes < need) { *why = "workspace too small for the row-epilogue exchange"; return cudaErrorInvalidValue; }
    // counters first, at an offset that depends on M only: row-epilogue launches of the same M
    // and any N (a layer's RESLN N = hidden and GELU N = ffn) share one workspace, and one
    // launch's float partials never land on another launch's counters
    uint8_t* w = reinterpret_cast<uint8_t*>(ws);
    const size_t nslot = (size_t)p.mblocks * p.ntn * 128, cnt_bytes = tc_counter_bytes(g.M) + tc_ksplit_bytes(g.M);
    p.xcnt = reinterpret_cast<unsigned*>(w);
    p.xstat = reinterpret_cast<float2*>(w + cnt_bytes);
    p.xamax = reinterpret_cast<float*>(w + cnt_bytes + nslot * 8);
    p.xmm = reinterpret_cast<float2*>(w + cnt_bytes + nslot * 12);
    p.yscr = KIND == EPI_GELU_Q4 ? reinterpret_cast<__half*>(w + cnt_bytes + nslot * 20) : nullptr;
    if (KIND == EPI_GELU_Q4 && Q4_GELU_DECOUPLED && (size_t)grid > tc_row_grid(g.M, g.N, TN)) {
      *why = "row-epilogue grid larger than the workspace sizing assumed";
      return cudaErrorInvalidValue;
    }
  }
  // CX: a single m-block whose ntn <= 16 CTAs can form one cluster exchanges its row partials
  // through distributed shared memory (the batch-1 row GEMMs without split-K)
  if constexpr ((KIND == EPI_GELU_Q4 || KIND == EPI_RESLN_Q4) && !PAIR && !SPLIT && TN <= 64) {
    if (p.mblocks == 1 && p.ntn <= 16 && p.ksplit == 1 && grid == p.ntn && tc_cx_enabled()) p.cx = 1;
  }
  note_launch();
  {
    cudaError_t le;
    if (p.cx) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = C::SMEM;
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)grid;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      le = cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
      if (le != cudaSuccess) {  // a cluster the GPU cannot place: the L2 rendezvous instead
        (void)cudaGetLastError();
        p.cx = 0;
      }
    }
    if (p.cx) {
      le = cudaSuccess;
    } else if constexpr (PAIR || SPLIT) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = C::SMEM;
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // SPLIT: the small-M latency path
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      static const bool no_pdl = prof_env("Q4_NO_PDL") != nullptr;  // profiling only
      cfg.numAttrs = (SPLIT && !no_pdl) ? 2 : 1;
      le = cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
    } else {
      le = launch_pdl(g.M <= kPdlMaxRows, kern, dim3(grid), dim3(THREADS), C::SMEM, s, ta, tb, p);
    }
    if (le != cudaSuccess) return le;
  }
  if (trace_path) {  // profiling only: dump the stamps of this launch (synchronous)
    static unsigned long long host[148 * 64 * 8];
    cudaMemcpy(host, trace_buf, sizeof(host), cudaMemcpyDeviceToHost);
    FILE* f = fopen(trace_path, "ab");
    if (f) {
      const int hdr[4] = {grid, KIND, TN, g.M};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
  }
  return cudaGetLastError();
}

// The R4 row kernel is off: measured slower (FFN1 253 vs 219 us, FFN2 243 vs 149 us at
// M = 32768; the pair N = 128 mainloop is shared-memory bound on the A unpack).  Q4_R4=1 in
// the profiling build selects it (A/B only).
bool tc_r4_enabled() {
  static const int env = [] { const char* e = prof_env("Q4_R4"); return e ? atoi(e) : 0; }();
  return env == 1;
}
constexpr int kR4MinRows = 8192;

// The CTA-pair mainloop is on by default where it measured faster; Q4_PAIR=0 disables it
// (profiling / A-B only).
bool tc_pair_enabled() {
  static const int env = [] { const char* e = prof_env("Q4_PAIR"); return e ? atoi(e) : -1; }();
  return env != 0;
}

// Split-K over a CTA cluster for the latency configs (M <= 512, TN = 64, >= 4 k-blocks): correct
// (the small-M parity tests pass through it) but measured slower -- BERT-base bs 1 per layer QKV
// 7.1 -> 9.7 us, O-proj 14.3 -> 18.1, FFN1 11.4 -> 14.4, FFN2 21.0 -> 21.5 (cluster prologue,
// shallower rings, the DSMEM reduction on the chain) -- so it is off; Q4_SPLIT=1 in the
// profiling build selects it (A/B only).
bool tc_split_enabled() {
  static const int env = [] { const char* e = prof_env("Q4_SPLIT"); return e ? atoi(e) : 0; }();
  return env == 1;
}

template <int TN, bool BI8, bool A8 = false>
cudaError_t run_tc_kind2(const GemmArgs& g, void* ws, size_t wsb, cudaStream_t s, const char** why) {
  if constexpr (TN == 64 && BI8) {
    if (!g.f16_ops && !g.a_zeros && !g.out_zeros && g.M <= 512 && g.K / 128 >= 4 && tc_split_enabled()) {
      switch (g.kind) {
        case EPI_I32: return run_tc<64, EPI_I32, true, A8, false, false, false, true>(g, ws, wsb, s, why);
        case EPI_F16: return run_tc<64, EPI_F16, true, A8, false, false, false, true>(g, ws, wsb, s, why);
        case EPI_GELU_Q4: return run_tc<64, EPI_GELU_Q4, true, A8, false, false, false, true>(g, ws, wsb, s, why);
        case EPI_RESLN_Q4: return run_tc<64, EPI_RESLN_Q4, true, A8, false, false, false, true>(g, ws, wsb, s, why);
      }
    }
  }
  if constexpr (A8) {
    if (!g.f16_ops && TN == 256 && g.M % 256 == 0 && g.M >= 8192 && (g.kind == EPI_F16 || g.kind == EPI_I32) &&
        g.N / TN <= num_sms() / 2 && g.mainloop != Q4_MAINLOOP_TCGEN05_W8_1CTA && tc_pair_enabled()) {  // W8A8 on the CTA-pair mainloop
      if (g.kind == EPI_I32) return run_tc<TN, EPI_I32, true, true, false, true>(g, ws, wsb, s, why);
      return run_tc<TN, EPI_F16, true, true, false, true>(g, ws, wsb, s, why);
    }
    if (g.f16_ops) {  // fp16 operands (q4_f16_linear): no I32 epilogue
      switch (g.kind) {
        case EPI_F16: return run_tc<TN, EPI_F16, true, true, true>(g, ws, wsb, s, why);
        case EPI_GELU_Q4: return run_tc<TN, EPI_GELU_Q4, true, true, true>(g, ws, wsb, s, why);
        case EPI_RESLN_Q4: return run_tc<TN, EPI_RESLN_Q4, true, true, true>(g, ws, wsb, s, why);
      }
      *why = "fp16 operands: no such epilogue";
      return cudaErrorInvalidValue;
    }
  }
  if constexpr (BI8 && !A8 && TN == 256) {
    // CTA-pair mainloop (cta_group::2) for large problems with prepacked weights
    // (F16 / I32 only: measured QKV 105.8 -> 95.4 us at M = 32768; the RESLN row epilogue
    // measured slower on pairs, 151 -> 160 us for FFN2, so it stays on the 1-CTA mainloop)
    if (g.M % 256 == 0 && g.M >= 8192 && (g.kind == EPI_F16 || g.kind == EPI_I32) && g.N / TN <= num_sms() / 2 && g.mainloop != Q4_MAINLOOP_TCGEN05_W8_1CTA &&
        tc_pair_enabled()) {
      if (g.kind == EPI_I32) return run_tc<TN, EPI_I32, true, false, false, true>(g, ws, wsb, s, why);
      return run_tc<TN, EPI_F16, true, false, false, true>(g, ws, wsb, s, why);
    }
  }
  switch (g.kind) {
    case EPI_I32: return run_tc<TN, EPI_I32, BI8, A8>(g, ws, wsb, s, why);
    case EPI_F16: return run_tc<TN, EPI_F16, BI8, A8>(g, ws, wsb, s, why);
    case EPI_GELU_Q4:
      if constexpr (!A8)
        if (g.a_zeros || g.out_zeros) return run_tc<TN, EPI_GELU_Q4, BI8, false, false, false, true>(g, ws, wsb, s, why);
      return run_tc<TN, EPI_GELU_Q4, BI8, A8>(g, ws, wsb, s, why);
    case EPI_RESLN_Q4:
      if constexpr (!A8)
        if (g.a_zeros || g.out_zeros) return run_tc<TN, EPI_RESLN_Q4, BI8, false, false, false, true>(g, ws, wsb, s, why);
      return run_tc<TN, EPI_RESLN_Q4, BI8, A8>(g, ws, wsb, s, why);
  }
  *why = "unknown epilogue kind";
  return cudaErrorInvalidValue;
}
template <int TN>
cudaError_t run_tc_kind(const GemmArgs& g, void* ws, size_t wsb, cudaStream_t s, const char** why) {
  if (g.a_i8) {
    if (!g.w_i8) { *why = "W8A8 needs int8 weight codes"; return cudaErrorInvalidValue; }
    return run_tc_kind2<TN, true, true>(g, ws, wsb, s, why);
  }
  if (g.w_i8) return run_tc_kind2<TN, true>(g, ws, wsb, s, why);
  return run_tc_kind2<TN, false>(g, ws, wsb, s, why);
}

}  // namespace

int tc_tile_n(int M, int N, int kind) {
  // Small M (latency configs): narrower tiles spread the work over more SMs.  Row
  // epilogues need >= 64 columns per tile (>= 16 code bytes per row per half).
  const bool row = kind == EPI_GELU_Q4 || kind == EPI_RESLN_Q4;
  static const int env_tn = prof_env("Q4_TN") ? atoi(prof_env("Q4_TN")) : 0;  // profiling only
  const int pref = env_tn ? env_tn : M <= 512 ? 64 : 256;
  static const int cand[] = {256, 128, 64, 32};
  for (int c : cand)
    if (c <= pref && N % c == 0 && !(row && c < 64)) return c;
  for (int c : cand)
    if (N % c == 0 && !(row && c < 64)) return c;
  return 0;
}

size_t tc_counter_bytes(int M) {
  const size_t mblocks = (size_t)(M + 127) / 128;
  return (4 * mblocks * sizeof(unsigned) + 255) & ~(size_t)255;
}

// Split-K over global reductions for the latency configs (M <= kKsplitMaxRows): slices of at
// least kKsplitMinKb k-blocks, as many as fit one CTA per SM next to the other tiles.
int tc_ksplit(int M, int N, int K, int TN, bool row) {
  // profiling only: Q4_KSPLIT forces the split (0 = off), Q4_KSPLIT_MINKB the k-loop threshold
  static const int env = prof_env("Q4_KSPLIT") && *prof_env("Q4_KSPLIT") ? atoi(prof_env("Q4_KSPLIT")) : -1;
  static const int minkb = prof_env("Q4_KSPLIT_MINKB") ? atoi(prof_env("Q4_KSPLIT_MINKB")) : kKsplitMinLoop;
  if (M <= 0 || M > kKsplitMaxRows || N > kKsplitMaxN || TN > 64 || env == 0) return 1;
  const int KB = (K + 127) / 128, tiles = ((M + 127) / 128) * (N / TN);
  if (KB < minkb) return 1;
  // a row epilogue that runs as one cluster (CX) is faster unsplit inside the layer (BERT-base
  // batch 1, 12 layers eager: FFN2 split 12 ways 0.608 ms, unsplit with CX 0.578 ms -- the 12
  // CTAs start under PDL while the previous kernel runs, 144 cannot)
  if (row && M <= 128 && N / TN <= 16 && tc_cx_enabled() && env < 0) return 1;
  int s = num_sms() / tiles;
  if (s > KB / kKsplitMinKb) s = KB / kKsplitMinKb;
  if (env > 1 && env <= KB && env * tiles <= num_sms()) s = env;
  return s >= 2 ? s : 1;
}
// The zero-at-rest split-K region after the rendezvous counters: [mblocks] x (tile counters |
// INT32 partials for N <= kKsplitMaxN); its offset and size depend on M only.
size_t tc_ksplit_bytes(int M) {
  if (M <= 0 || M > kKsplitMaxRows) return 0;
  const size_t mblocks = (size_t)(M + 127) / 128;
  return mblocks * (kKsplitCntBytes + (size_t)kKsplitMaxN * 128 * 4);
}

// CTAs of a row-epilogue launch (the grid run_tc picks): groups of ntn co-resident CTAs
size_t tc_row_grid(int M, int N, int TN) {
  const size_t mblocks = (size_t)(M + 127) / 128, ntn = (size_t)N / TN;
  size_t groups = ntn ? (size_t)num_sms() / ntn : 0;
  if (groups > mblocks) groups = mblocks;
  return groups * ntn;
}

size_t tc_workspace_bytes(int M, int N, int TN, int kind) {
  if (TN <= 0) return 0;
  if (kind != EPI_GELU_Q4 && kind != EPI_RESLN_Q4) {
    const size_t k = tc_ksplit_bytes(M);
    return k ? tc_counter_bytes(M) + k : 0;  // F16 / I32: the split-K region only
  }
  // partial slots for ntn = N / min(TN, 128): the R4 row kernel (TN = 128) may run instead
  const size_t mblocks = (size_t)(M + 127) / 128, ntn = (size_t)N / (TN < 128 ? TN : 128);
  size_t b = tc_counter_bytes(M) + tc_ksplit_bytes(M) + mblocks * ntn * 128 * 20;  // stats (8) | amax (4) | asym min/max (8)
  // GELU_Q4: two y parking slots per epilogue group (pass B of tile t runs after pass A of t + 2)
  if (kind == EPI_GELU_Q4 && Q4_GELU_DECOUPLED) b += tc_row_grid(M, N, TN) * 4 * 128 * (size_t)TN * 2;
  return b;
}

cudaError_t launch_w4a4_tc(const GemmArgs& g, void* ws, size_t ws_bytes, cudaStream_t s, const char** why) {
  if (g.M == 0) return cudaSuccess;
  // Row epilogues at large M with prepacked weights: the R4 pair kernel (four accumulators)
  if ((g.kind == EPI_GELU_Q4 || g.kind == EPI_RESLN_Q4) && g.w_i8 && !g.a_i8 && !g.f16_ops && !g.a_zeros &&
      g.M % 256 == 0 && g.M >= kR4MinRows && g.N % 128 == 0 && g.mainloop != Q4_MAINLOOP_TCGEN05_W8_1CTA &&
      tc_pair_enabled() && tc_r4_enabled()) {
    if (g.kind == EPI_GELU_Q4) return run_tc<128, EPI_GELU_Q4, true, false, false, true>(g, ws, ws_bytes, s, why);
    return run_tc<128, EPI_RESLN_Q4, true, false, false, true>(g, ws, ws_bytes, s, why);
  }
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

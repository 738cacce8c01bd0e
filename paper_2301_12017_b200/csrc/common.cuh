// common.cuh -- sm_100a PTX wrappers shared by the kernels of the CUDA path
// (mbarrier, TMA, tcgen05/TMEM, cluster/DSMEM, fp16 packing).  Product code only;
// nothing here is shared with the CPU oracle.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#define Q4_DEV __device__ __forceinline__

namespace q4 {

Q4_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ------------------------------------------------------------------ mbarrier
Q4_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
Q4_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
Q4_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
Q4_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the phase completes
// (or the hint expires) instead of spinning and stealing issue slots from working warps.
Q4_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(0x989680u)
      : "memory");
  return ok != 0;
}
// Wait with cluster-scope acquire (barriers that receive arrivals from the peer CTA of a pair).
Q4_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
Q4_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels launched with launch_pdl() start their prologue (barrier init, TMEM alloc,
// descriptor prefetch) while the previous kernel in the stream drains, and must execute
// pdl_wait() before touching any global memory another kernel produces or consumes.
Q4_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
Q4_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ proxies / fences
Q4_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ TMA
Q4_DEV void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 2-D tiled load: box at (c0 = innermost coordinate, c1 = row) -> smem, completes tx on bar.
Q4_DEV void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Same, with an L2 cache-policy hint (policy from l2_policy_evict_*).
Q4_DEV void tma_load_2d_hint(void* smem_dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1,
                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
Q4_DEV uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
Q4_DEV uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
Q4_DEV void st_global_hint(void* ptr, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(policy)
               : "memory");
}

// ------------------------------------------------------------------ cluster
Q4_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
Q4_DEV void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
Q4_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
Q4_DEV void cluster_sync() { cluster_arrive(); cluster_wait(); }
// Map a local smem address to the same offset in CTA `rank` of the cluster.
Q4_DEV uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
Q4_DEV void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
Q4_DEV void st_cluster_v2f32(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

// ------------------------------------------------------------------ tcgen05 / TMEM
Q4_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
Q4_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
Q4_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
Q4_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32, cta_group::1.
Q4_DEV void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05 ops of this thread complete.
Q4_DEV void umma_f16kk(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
Q4_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
Q4_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
Q4_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 columns of 32-bit: thread i of the warp gets lane (base_lane + i), cols c..c+31.
Q4_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
Q4_DEV void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
Q4_DEV void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
Q4_DEV void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}

// ------------------------------------------------------------------ UMMA descriptors
// Shared-memory matrix descriptor (sm100 "version 1"), K-major, swizzled canonical
// layout: 8-row atoms of `pitch` bytes, atoms SBO bytes apart.
//   layout: 2 = SWIZZLE_128B (pitch 128), 4 = SWIZZLE_64B (pitch 64)
Q4_DEV uint64_t umma_smem_desc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;                             // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;     // SBO
  d |= (uint64_t)1 << 46;                               // version = 1 (Blackwell)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}
// Instruction descriptor for kind::f16: f16 x f16 -> f32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_f16kk(int M, int N) {
  return (1u << 4)  // c_format = F32 (a_format = b_format = F16: 0)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// Instruction descriptor for kind::i8: s8 x s8 -> s32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_i8(int M, int N) {
  return (2u << 4)                 // c_format = S32
         | (1u << 7)               // a_format = signed 8-bit
         | (1u << 10)              // b_format = signed 8-bit
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------------ small math
Q4_DEV uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
Q4_DEV float2 unpack_half2(uint32_t u) {
  __half2 h = *reinterpret_cast<__half2*>(&u);
  return __half22float2(h);
}
// Exact symmetric INT4 code of fp16 value y (as float) given row amax a > 0:
// rint(div.rn(7y, a)) == round-half-even of the exact rational 7y/a for all fp16 pairs.
Q4_DEV int q4_code(float y, float a) { return __float2int_rn(__fdiv_rn(7.0f * y, a)); }

// The same code, fast: with r7 = RN(7/a), p = y*r7 is within 1e-6 of 7y/a (|y| <= a), so
// p's nearest integer is the answer unless p is within 2e-6 of a half-integer; there the
// side is decided exactly by the sign of t - a*h (t = 7y, h = that half-integer; both are
// short fp16 x small-integer products, so the FMA result is exact).  Half-even ties.
Q4_DEV int requant_code(float y, float a, float r7) {
  const float p = y * r7;
  const float s = p + 12582912.0f;  // 1.5 * 2^23: rounds p to an integer, half to even
  const float fn = s - 12582912.0f;
  int n = __float_as_int(s) - 0x4B400000;
  const float d0 = p - fn;
  if (fabsf(d0) > 0.499998f) {
    const float h = fn + copysignf(0.5f, d0);
    const float e = fmaf(-a, h, 7.0f * y);
    const int lo = (int)floorf(h), hi = lo + 1;
    n = e > 0.f ? hi : (e < 0.f ? lo : ((lo & 1) ? hi : lo));
  }
  return n;
}
// Two INT4 codes -> low byte, previous word shifted left by 8 (I2IP, saturating).
Q4_DEV uint32_t cvt_pack_s4(int hi, int lo, uint32_t prev) {
  uint32_t d;
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(hi), "r"(lo), "r"(prev));
  return d;
}
// 8 fp16 values (4 packed words) -> 8 codes packed in one word (element i at bits 4i).
// amax <= 0 gives all-zero codes (R5).  y is clamped to [-clip, clip] when clip > 0.
Q4_DEV uint32_t requant8(const uint32_t (&h)[4], float amax, float r7, float clip) {
  if (!(amax > 0.f)) return 0u;
  float y[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h[j]));
    y[2 * j] = f.x;
    y[2 * j + 1] = f.y;
  }
  if (clip > 0.f) {
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = fminf(fmaxf(y[j], -clip), clip);
  }
  int q[8];
  float dmax = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float p = y[j] * r7;
    const float sm = p + 12582912.0f;
    dmax = fmaxf(dmax, fabsf(p - (sm - 12582912.0f)));
    q[j] = __float_as_int(sm) - 0x4B400000;
  }
  if (dmax > 0.499998f) {
#pragma unroll
    for (int j = 0; j < 8; ++j) q[j] = requant_code(y[j], amax, r7);
  }
  uint32_t w = cvt_pack_s4(q[7], q[6], 0u);
  w = cvt_pack_s4(q[5], q[4], w);
  w = cvt_pack_s4(q[3], q[2], w);
  return cvt_pack_s4(q[1], q[0], w);
}
// Pack 8 codes (each in [-8,7]) into a 32-bit word, element i in bits [4i, 4i+4).
Q4_DEV uint32_t pack8(const int (&q)[8]) {
  uint32_t w = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) w |= ((uint32_t)q[i] & 0xFu) << (4 * i);
  return w;
}
// The K-permutation unpack: a 32-bit word of 8 packed
// nibbles -> two words of 4 int8 each holding 16*q.  lo: elements 0,2,4,6; hi: 1,3,5,7.
Q4_DEV uint32_t nib_lo16(uint32_t w) { return (w << 4) & 0xF0F0F0F0u; }
Q4_DEV uint32_t nib_hi16(uint32_t w) { return w & 0xF0F0F0F0u; }

Q4_DEV float gelu_erf(float t) { return 0.5f * t * (1.0f + erff(t * 0.70710678118654752f)); }

// ------------------------------------------------------------------ packed fp32x2 (FFMA2 etc.)
Q4_DEV float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
Q4_DEV float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
Q4_DEV float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
Q4_DEV float2 f2(float v) { return make_float2(v, v); }
Q4_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// (p.x - h.lo, p.y - h.hi) with the fp16 halves of h taken as exact f32 (FHFMA: f16*f16+f32,
// one rounding -> exact when h = fp16(p)).
Q4_DEV float2 sub_half2_f32(uint32_t h, float2 p) {
  float2 d;
  asm("{.reg .f16 a, b, m;\n\tmov.b32 {a, b}, %2;\n\tmov.b16 m, 0xBC00;\n\t"
      "fma.rn.f32.f16 %0, a, m, %3;\n\tfma.rn.f32.f16 %1, b, m, %4;}"
      : "=f"(d.x), "=f"(d.y)
      : "r"(h), "f"(p.x), "f"(p.y));
  return d;
}
// (p.x + h.lo, p.y + h.hi) with the fp16 halves of h taken as exact f32 (FHFMA h*1+p:
// one rounding, the same result as converting h and adding).
Q4_DEV float2 add_half2_f32(uint32_t h, float2 p) {
  float2 d;
  asm("{.reg .f16 a, b, m;\n\tmov.b32 {a, b}, %2;\n\tmov.b16 m, 0x3C00;\n\t"
      "fma.rn.f32.f16 %0, a, m, %3;\n\tfma.rn.f32.f16 %1, b, m, %4;}"
      : "=f"(d.x), "=f"(d.y)
      : "r"(h), "f"(p.x), "f"(p.y));
  return d;
}
Q4_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// requant8(h, amax, r7, 0) with packed fp32x2 arithmetic, for amax > 0 and |y| <= amax,
// split into a branch-free stage and a rare fix-up so several words can be in flight.
// s = p + 1.5*2^23 holds round-half-even(p) = n in [-7, 7] as bits 0x4B400000 + n, so the
// low byte of s is n in two's complement: gather the 8 low bytes with PRMT and merge the
// nibbles (even elements low, odd high) instead of subtracting and packing per element.
// Returns the packed word; dmax collects max |p - rint(p)| (> 0.499998: use requant8).
Q4_DEV uint32_t requant8_nofix(const uint32_t (&h)[4], float r7, float& dmax) {
  uint32_t sb[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 p = fmul2(unpack_half2(h[j]), f2(r7));
    const float2 sm = fadd2(p, f2(12582912.0f));
    const float2 d = ffma2(fadd2(sm, f2(-12582912.0f)), f2(-1.f), p);  // exact p - rint(p)
    dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
    sb[2 * j] = __float_as_uint(sm.x);
    sb[2 * j + 1] = __float_as_uint(sm.y);
  }
  const uint32_t ev = prmt(prmt(sb[0], sb[2], 0x40u), prmt(sb[4], sb[6], 0x40u), 0x5410u);
  const uint32_t od = prmt(prmt(sb[1], sb[3], 0x40u), prmt(sb[5], sb[7], 0x40u), 0x5410u);
  return (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
}

// ------------------------------------------------------------------ 8-bit codes (W8A8)
// The same quantizer at b = 8 bits (qmax = 127; oracle O-11): n = rhe(127 y / amax).
// p = y * RN(127/amax) differs from the exact 127 y / amax by <= 127 * 2^-23 < 1.6e-5, so
// rint(p) is exact unless p is within 1e-4 of a half-integer; there the exact FMA
// tie-break decides (127 y and amax * h are exact in the fma: 18- and 20-bit products).
Q4_DEV int requant_code_i8(float y, float a, float rq) {
  const float p = y * rq;
  const float s = p + 12582912.0f;
  const float fn = s - 12582912.0f;
  int n = __float_as_int(s) - 0x4B400000;
  const float d0 = p - fn;
  if (fabsf(d0) > 0.4999f) {
    const float h = fn + copysignf(0.5f, d0);
    const float e = fmaf(-a, h, 127.0f * y);
    const int lo = (int)floorf(h), hi = lo + 1;
    n = e > 0.f ? hi : (e < 0.f ? lo : ((lo & 1) ? hi : lo));
  }
  return n;
}
// 8 fp16 values (4 packed words) -> 8 int8 codes (2 words, element i in byte i).  The low
// byte of s = p + 1.5*2^23 is rint(p) in two's complement; PRMT gathers the bytes.
Q4_DEV uint2 requant8_i8(const uint32_t (&h)[4], float amax, float rq, float clip) {
  if (!(amax > 0.f)) return make_uint2(0u, 0u);
  float2 y[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    y[j] = unpack_half2(h[j]);
    if (clip > 0.f) y[j] = make_float2(fminf(fmaxf(y[j].x, -clip), clip), fminf(fmaxf(y[j].y, -clip), clip));
  }
  uint32_t sb[8];
  float dmax = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 p = fmul2(y[j], f2(rq));
    const float2 sm = fadd2(p, f2(12582912.0f));
    const float2 d = ffma2(fadd2(sm, f2(-12582912.0f)), f2(-1.f), p);
    dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
    sb[2 * j] = __float_as_uint(sm.x);
    sb[2 * j + 1] = __float_as_uint(sm.y);
  }
  if (dmax > 0.4999f) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sb[2 * j] = (uint32_t)requant_code_i8(y[j].x, amax, rq);
      sb[2 * j + 1] = (uint32_t)requant_code_i8(y[j].y, amax, rq);
    }
  }
  return make_uint2(prmt(prmt(sb[0], sb[1], 0x40u), prmt(sb[2], sb[3], 0x40u), 0x5410u),
                    prmt(prmt(sb[4], sb[5], 0x40u), prmt(sb[6], sb[7], 0x40u), 0x5410u));
}

// GELU (erf form, reading R11) for two values, ~12 ops/element, |err| <= 5e-6 vs fp64
// (float32 evaluation, scripts/fit_gelu.py):
// GELU(x) = max(x,0) - |x| Q(|x|) with Q the normal upper tail, Q(t) = exp(-t^2/2) R(t) and
// R a degree-8 polynomial in v = 2.75 - min(t, 5.5) (least squares weighted by the GELU
// error t exp(-t^2/2), iteratively reweighted towards minimax; for t > 5.5, |x| Q < 1e-7).
// One MUFU.EX2 per element; everything else is FFMA2/FMUL2.
Q4_DEV float2 gelu2(float2 t) {
  const float2 tn = make_float2(fmaxf(-fabsf(t.x), -5.5f), fmaxf(-fabsf(t.y), -5.5f));  // -min(|t|, 5.5)
  const float2 v = fadd2(tn, f2(2.75f));
  float2 r = f2(1.111536767e-05f);
  r = ffma2(r, v, f2(-5.116840384e-06f));
  r = ffma2(r, v, f2(-6.360232419e-06f));
  r = ffma2(r, v, f2(3.042680910e-04f));
  r = ffma2(r, v, f2(7.307167980e-04f));
  r = ffma2(r, v, f2(2.832866041e-03f));
  r = ffma2(r, v, f2(1.117350161e-02f));
  r = ffma2(r, v, f2(3.947244585e-02f));
  r = ffma2(r, v, f2(1.307167113e-01f));
  const float2 ea = fmul2(fmul2(tn, tn), f2(-0.72134752044448170f));  // -t^2/2 * log2(e)
  const float2 qv = fmul2(make_float2(ex2_approx(ea.x), ex2_approx(ea.y)), r);
  return ffma2(tn, qv, make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f)));
}

// tcgen05.wait::ld that also carries the loaded registers as operands, so no use of them can be
// scheduled above the wait (software-pipelined TMEM loads)
Q4_DEV void tmem_wait_ld_dep(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}

// GELU (erf form, reading R11) of 16 dequantized accumulators, t = acc sa sw + b, as 8 packed fp16
// pairs.  GELU(x) = max(x,0) + tn Q(|x|)-ish with tn = -min(|x|, 4.5): Q(t) = exp(-t^2/2) R(u),
// R a degree-6 polynomial in u = tn + 2.25 (scripts/fit_gelu.py 4.5 6: |err| <= 4.1e-5 against
// the fp64 erf form in this float32 evaluation order, 1/24 of the 1e-3 absolute parity budget).
// The 8 pairs advance in lockstep, one Horner step for all of them at a time: 8 independent
// chains per step instead of the compiler's register-bound interleave.
// ASYM (asymmetric activations, O-16): t = sw (sa acc + za colsum) + b with the per-column
// weight-code sums at `cs`.
template <bool FACC, bool ASYM = false>
Q4_DEV void gelu16(const uint32_t (&v)[16], float2 sa2, const float* sw, const float* bs, uint32_t (&h)[8],
                   float2 za2 = make_float2(0.f, 0.f), const float* cs = nullptr) {
  constexpr float HI = 4.5f, H2 = 2.25f;
  const float4* pw = reinterpret_cast<const float4*>(sw);
  const float4* pb = reinterpret_cast<const float4*>(bs);
  float2 t[8], u[8], r[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 w = pw[j], bb = pb[j];
    const float2 a0 = FACC ? make_float2(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]))
                           : make_float2((float)(int)v[4 * j], (float)(int)v[4 * j + 1]);
    const float2 a1 = FACC ? make_float2(__uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]))
                           : make_float2((float)(int)v[4 * j + 2], (float)(int)v[4 * j + 3]);
    if constexpr (ASYM) {
      const float4 c = reinterpret_cast<const float4*>(cs)[j];
      t[2 * j] = ffma2(ffma2(a0, sa2, fmul2(za2, make_float2(c.x, c.y))), make_float2(w.x, w.y), make_float2(bb.x, bb.y));
      t[2 * j + 1] = ffma2(ffma2(a1, sa2, fmul2(za2, make_float2(c.z, c.w))), make_float2(w.z, w.w),
                           make_float2(bb.z, bb.w));
    } else {
      t[2 * j] = ffma2(fmul2(a0, sa2), make_float2(w.x, w.y), make_float2(bb.x, bb.y));
      t[2 * j + 1] = ffma2(fmul2(a1, sa2), make_float2(w.z, w.w), make_float2(bb.z, bb.w));
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    u[j] = fadd2(make_float2(fmaxf(-fabsf(t[j].x), -HI), fmaxf(-fabsf(t[j].y), -HI)), f2(H2));
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = ffma2(f2(2.548979828e-04f), u[j], f2(4.253684019e-04f));
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = ffma2(r[j], u[j], f2(7.912631845e-04f));
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = ffma2(r[j], u[j], f2(5.301531870e-03f));
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = ffma2(r[j], u[j], f2(1.732770912e-02f));
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = ffma2(r[j], u[j], f2(5.303432420e-02f));
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = ffma2(r[j], u[j], f2(1.536411792e-01f));
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 tn = fadd2(u[j], f2(-H2));
    const float2 ea = fmul2(fmul2(tn, tn), f2(-0.72134752044448170f));  // -t^2/2 * log2(e)
    const float2 qv = fmul2(make_float2(ex2_approx(ea.x), ex2_approx(ea.y)), r[j]);
    const float2 y = ffma2(tn, qv, make_float2(fmaxf(t[j].x, 0.f), fmaxf(t[j].y, 0.f)));
    h[j] = pack_half2(y.x, y.y);
  }
}

// Asymmetric INT4 code of fp16 value x (as float) given the row min mn and D = max - min > 0
// (NEXT-3, oracle O-15; readings R17/R18): q = rhe(15 (x - mn) / D) in [0, 15].  x - mn and D
// are differences of fp16 values, exact in fp64 (<= 41 significant bits), so p = d * (15/D) is
// within 1e-14 of the rational; near a half-integer the exact residual 15 d - D h decides.
Q4_DEV uint32_t asym_code(float x, double mn, double D, double r15) {
  const double d = (double)x - mn;
  const double p = d * r15;
  double n = rint(p);
  if (fabs(p - n) > 0.4999999) {
    const double h = floor(p) + 0.5;
    const double e = fma(-D, h, 15.0 * d);
    n = e > 0.0 ? h + 0.5 : (e < 0.0 ? h - 0.5 : (fmod(h - 0.5, 2.0) == 0.0 ? h - 0.5 : h + 0.5));
  }
  return (uint32_t)(int)fmin(n, 15.0);
}
// 8 fp16 values (4 packed words) -> 8 asymmetric codes in one word (element i at bits 4i);
// D <= 0 (constant row) gives all-zero codes.  Fast path in fp32: d = x - mn and p = d * fl(15/D)
// carry a relative error <= 3 * 2^-24, so |p - p_exact| <= 15 * 1.8e-7 < 3e-6 and rint(p) is the
// exact code unless p is within 1e-5 of a half-integer; those 8-value chunks take asym_code's
// exact fp64 residual path.
Q4_DEV uint32_t requant8_asym(const uint32_t (&h)[4], float mn, float mx) {
  const double D = (double)mx - (double)mn;
  if (!(D > 0.0)) return 0u;
  const float r15f = (float)(15.0 / D);
  const float2 mn2 = f2(-mn), r2 = f2(r15f);
  uint32_t w = 0;
  float dmax = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 p = fmul2(fadd2(unpack_half2(h[j]), mn2), r2);
    const float2 sm = fadd2(p, f2(12582912.0f));                  // rint(p) in the low bits
    const float2 d = ffma2(fadd2(sm, f2(-12582912.0f)), f2(-1.f), p);  // p - rint(p)
    dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
    const uint32_t c0 = min((uint32_t)(__float_as_int(sm.x) - 0x4B400000), 15u);
    const uint32_t c1 = min((uint32_t)(__float_as_int(sm.y) - 0x4B400000), 15u);
    w |= (c0 | (c1 << 4)) << (8 * j);
  }
  if (dmax > 0.49999f) {
    const double r15 = 15.0 / D, m = (double)mn;
    w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_half2(h[j]);
      w |= asym_code(f.x, m, D, r15) << (8 * j);
      w |= asym_code(f.y, m, D, r15) << (8 * j + 4);
    }
  }
  return w;
}

}  // namespace q4

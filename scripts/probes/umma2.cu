// Profiling / design probe (not part of the product): one 256 x 256 x K int8 tile on a CTA
// pair with tcgen05.mma.cta_group::2 (M = 256: each CTA holds 128 rows of A and 128 rows of
// the K-major B, the leader issues the MMA, both CTAs' TMA loads complete on the leader's
// mbarrier, the commit multicasts to both CTAs).  Checks the INT32 result against the CPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I ../../paper_2301_12017_b200/csrc umma2.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"

using namespace q4;

constexpr int KB_BYTES = 128, ROWS = 128, ST = 2;
constexpr int A_ST = ROWS * KB_BYTES, B_ST = ROWS * KB_BYTES, STAGE = A_ST + B_ST;
constexpr int SMEM = ST * STAGE + 1024 + 256;

__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  unsigned n = 0;
  while (!mbar_try_wait(a, parity))
    if (++n > (1u << 24)) __trap();
}
__device__ __forceinline__ void tma_load_2sm(uint32_t dst, const void* tmap, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0),
      "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma2_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    umma2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                 int32_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int KBN = K / 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    // both CTAs: own half of A (rows 128 rank ..) and of B (N rows 128 rank ..) -> own smem;
    // completion counted on the leader's full barrier
    for (int kb = 0; kb < KBN; ++kb) {
      const int s = kb % ST;
      wait_bounded(&empty[s], ((kb / ST) & 1u) ^ 1u);
      const uint32_t lead_full = mapa(smem_u32(&full[s]), 0);
      if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE);
      uint8_t* st = smem + s * STAGE;
      tma_load_2sm(smem_u32(st), &tmA, lead_full, kb * 128, 128 * rank);
      tma_load_2sm(smem_u32(st + A_ST), &tmB, lead_full, kb * 128, 128 * rank);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    for (int kb = 0; kb < KBN; ++kb) {
      const int s = kb % ST;
      wait_bounded(&full[s], (kb / ST) & 1u);
      tc_fence_after();
      const uint32_t ua = smem_u32(smem + s * STAGE), ub = ua + A_ST;
      for (int ks = 0; ks < 4; ++ks)
        umma2_i8(tmem, umma_smem_desc(ua + ks * 32, 1024, 2), umma_smem_desc(ub + ks * 32, 1024, 2), idesc,
                 (kb | ks) != 0);
      commit2_mc(&empty[s]);
    }
    commit2_mc(tfull);
  } else if (warp >= 2) {
    const int q = warp & 3;  // TMEM lane quarter of this warp
    wait_bounded(tfull, 0);
    tc_fence_after();
    const int row = 128 * rank + 32 * q + lane;
    for (int c = 0; c < 256; c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + c, v);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) out[row * 256 + c + i] = (int32_t)v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int M = 256, N = 256, K = 512;
  std::vector<int8_t> A(M * K), B(N * K);
  srand(1);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dO;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
  cudaMemset(dO, 0, M * N * 4);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  EncFn enc = (EncFn)p;
  CUtensorMap ta, tb;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M}, str[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  dims[1] = N;
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(umma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  umma2_kernel<<<2, 192, SMEM>>>(ta, tb, K, dO);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int32_t> O(M * N);
  cudaMemcpy(O.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[m * K + k] * B[n * K + k];
      if (s != O[m * N + n] && bad++ < 5) printf("mismatch (%d,%d): %d vs %ld\n", m, n, O[m * N + n], s);
    }
  printf("mismatches: %ld of %d\n", bad, M * N);
  return bad != 0;
}

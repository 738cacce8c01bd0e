// Design probe (not part of the product): tcgen05.mma.sp.cta_group::1.kind::i8 on one CTA
// (SURVEY 8(f) NEXT-4, 2:4-sparse weights).  A = W [128 x 128] 2:4-sparse int8 (compressed:
// [128 x 64] values + metadata in TMEM), B = X [128 x 128] dense int8, D[n][m] = sum_k W[n][k]
// X[m][k] in TMEM.  Operands are written into shared memory in the SWIZZLE_128B K-major layout
// by plain stores (no TMA), the metadata into TMEM with tcgen05.st.  Tries metadata
// placements / encodings and reports the mismatch count of each against the CPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I ../../paper_2301_12017_b200/csrc umma_sp.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"

using namespace q4;

constexpr int R = 128, KL = 128;  // rows (channels / tokens), logical K
constexpr int A_BYTES = R * 128, B_BYTES = R * 128;
constexpr int SMEM = A_BYTES + B_BYTES + 1024 + 256;

__device__ __forceinline__ void umma_sp(uint32_t d, uint64_t a, uint64_t b, uint32_t e, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %5, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(e),
      "r"(acc), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}

// variant: bit 0 = metadata address per MMA (0: +2 columns per MMA, 1: same address + id2 = ks)
__global__ void __launch_bounds__(128, 1) sp_kernel(const uint8_t* Wc, const uint32_t* meta, const int8_t* X,
                                                   int32_t* out, int variant) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint8_t* sa = smem;
  uint8_t* sb = smem + A_BYTES;
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + A_BYTES + B_BYTES);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // A: compressed rows of 64 bytes placed in 128-byte SWIZZLE_128B rows (bytes 64..127 unused)
  for (int r = 0; r < R; ++r)
    if (t < 8) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (t < 4) v = *reinterpret_cast<const uint4*>(Wc + r * 64 + 16 * t);
      *reinterpret_cast<uint4*>(sa + r * 128 + ((t ^ (r & 7)) << 4)) = v;
    }
  for (int r = 0; r < R; ++r)
    if (t < 8) *reinterpret_cast<uint4*>(sb + r * 128 + ((t ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(X + r * KL + 16 * t);
  if (t == 0) { mbar_init(done, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(tslot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // metadata: lane = row n, 4 words (2 MMAs x 64 bits) at columns 128..131
  {
    uint32_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = meta[(32 * warp + lane) * 4 + i];
    tmem_st4(tmem + ((uint32_t)(32 * warp) << 16) + 128, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint32_t idesc0 = umma_idesc_i8(128, 128) | (1u << 2);
    for (int ks = 0; ks < 2; ++ks) {  // logical K = 64 per MMA: 32 compressed bytes of A, 64 bytes of B
      const uint32_t e = (variant & 1) ? tmem + 128 : tmem + 128 + 2 * ks;
      const uint32_t idesc = (variant & 1) ? (idesc0 | (uint32_t)ks) : idesc0;
      umma_sp(tmem, umma_smem_desc(smem_u32(sa) + ks * 32, 1024, 2), umma_smem_desc(smem_u32(sb) + ks * 64, 1024, 2),
              e, idesc, ks != 0);
    }
    umma_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out[(32 * warp + lane) * 128 + c + i] = (int32_t)v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<int8_t> W(R * KL, 0), X(R * KL);
  std::vector<int> idx(R * KL / 2);
  srand(7);
  for (int n = 0; n < R; ++n)
    for (int g = 0; g < KL / 4; ++g) {
      int i0 = rand() % 4, i1 = rand() % 4;
      while (i1 == i0) i1 = rand() % 4;
      if (i0 > i1) { int tt = i0; i0 = i1; i1 = tt; }
      W[n * KL + 4 * g + i0] = (int8_t)(rand() % 15 - 7);
      W[n * KL + 4 * g + i1] = (int8_t)(rand() % 15 - 7);
      idx[n * (KL / 2) + 2 * g] = i0;
      idx[n * (KL / 2) + 2 * g + 1] = i1;
    }
  for (auto& x : X) x = (int8_t)(rand() % 15 - 7);
  std::vector<uint8_t> Wc(R * 64);
  for (int n = 0; n < R; ++n)
    for (int j = 0; j < 64; ++j) Wc[n * 64 + j] = (uint8_t)W[n * KL + 4 * (j / 2) + idx[n * 64 + j]];
  // metadata encodings: per row 32 groups x 4 bits = 128 bits = 4 words
  // enc 0: group g -> bits [4g, 4g+4) = i0 | i1 << 2 ; enc 1: i1 | i0 << 2
  uint8_t *dWc;
  uint32_t* dM;
  int8_t* dX;
  int32_t* dO;
  cudaMalloc(&dWc, R * 64); cudaMalloc(&dM, R * 16); cudaMalloc(&dX, R * KL); cudaMalloc(&dO, R * R * 4);
  cudaMemcpy(dWc, Wc.data(), R * 64, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), R * KL, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(sp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  for (int enc = 0; enc < 2; ++enc)
    for (int variant = 0; variant < 2; ++variant) {
      std::vector<uint32_t> M(R * 4, 0);
      for (int n = 0; n < R; ++n)
        for (int g = 0; g < 32; ++g) {
          int i0 = idx[n * 64 + 2 * g], i1 = idx[n * 64 + 2 * g + 1];
          uint32_t nib = enc == 0 ? (uint32_t)(i0 | (i1 << 2)) : (uint32_t)(i1 | (i0 << 2));
          M[n * 4 + g / 8] |= nib << (4 * (g % 8));
        }
      cudaMemcpy(dM, M.data(), R * 16, cudaMemcpyHostToDevice);
      cudaMemset(dO, 0, R * R * 4);
      sp_kernel<<<1, 128, SMEM>>>(dWc, dM, dX, dO, variant);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<int32_t> O(R * R);
      cudaMemcpy(O.data(), dO, R * R * 4, cudaMemcpyDeviceToHost);
      long bad = 0;
      for (int n = 0; n < R; ++n)
        for (int m = 0; m < R; ++m) {
          long s = 0;
          for (int k = 0; k < KL; ++k) s += (long)W[n * KL + k] * X[m * KL + k];
          if (s != O[n * R + m]) ++bad;
        }
      printf("enc %d variant %d: %s, mismatches %ld of %d\n", enc, variant, cudaGetErrorString(e), bad, R * R);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}

// Microbenchmark: latency of tcgen05.ld (32x32b.x{8,16,32}) + tcgen05.wait::ld, and of
// tcgen05.st + wait::st, for 1 and 4 warps per CTA.  Prints cycles per round trip.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int X>
__global__ void k(unsigned long long* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = i;
  unsigned long long acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (X == 32) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]) : "r"(t + (it & 7) * 32));
    } else {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "r"(t + (it & 7) * 8));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    acc += v[0] + v[7];
  }
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "r"(t + (it & 7) * 8), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  long long t2 = clock64();
  if ((threadIdx.x & 31) == 0) { out[warp * 3] = (t1 - t0) / iters; out[warp * 3 + 1] = (t2 - t1) / iters; out[warp * 3 + 2] = acc; }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64 * 8); unsigned long long h[64];
  for (int w : {1, 4, 8}) {
    k<32><<<1, 32 * w>>>(d, 1000); cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
    printf("warps=%d x32: ld+wait %llu cyc, st8+wait %llu cyc\n", w, h[0], h[1]);
    k<8><<<1, 32 * w>>>(d, 1000); cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
    printf("warps=%d x8 : ld+wait %llu cyc, st8+wait %llu cyc\n", w, h[0], h[1]);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}

#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out) {
  int a = 3, b = -2; uint32_t c = 0x12345678u;
  uint32_t d;
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  out[0] = d;
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(9), "r"(-9), "r"(0u));
  out[1] = d;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  out[2] = d;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 16); k<<<1,1>>>(d); uint32_t h[4]; cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
  printf("s4(a=3,b=-2,c=0x12345678) = 0x%08x\ns4(9,-9,0) = 0x%08x\ns8(3,-2,c) = 0x%08x\n", h[0], h[1], h[2]);
}

// Profiling probe (not part of the product): throughput of I2FP.F32.S32, F2FP.F16.F32.PACK_AB,
// MUFU.EX2 and FFMA2-class ops per SM, to see which epilogue conversions share the XU pipe.
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k_i2f(int* out, int n) {
  int a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  float s = 0.f;
  for (int i = 0; i < n; ++i) {
    s += (float)a + (float)b + (float)c + (float)d;
    a += 1; b += 3; c += 5; d += 7;
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = (int)s;
}
__global__ void k_ex2(int* out, int n) {
  float a = threadIdx.x * 1e-3f, b = a + 1, c = a + 2, d = a + 3;
  for (int i = 0; i < n; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = (int)(a + b + c + d);
}
__global__ void k_f2h(int* out, int n) {
  float a = threadIdx.x * 1e-3f, b = a + 1, c = a + 2, d = a + 3;
  unsigned acc = 0;
  for (int i = 0; i < n; ++i) {
    __half2 h0 = __floats2half2_rn(a, b), h1 = __floats2half2_rn(c, d);
    acc ^= *reinterpret_cast<unsigned*>(&h0) + *reinterpret_cast<unsigned*>(&h1);
    a += 1.f; b += 1.f; c += 1.f; d += 1.f;
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = (int)acc;
}
__global__ void k_iadd(int* out, int n) {
  int a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  for (int i = 0; i < n; ++i) {
    a = (a >> 1) + b; b = (b >> 1) + c; c = (c >> 1) + d; d = (d >> 1) + a;
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = a ^ b ^ c ^ d;
}
int main() {
  int* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 1 << 14;
  const char* names[] = {"I2F (4 per iter)", "MUFU.EX2 (4)", "F2F pack (2 cvt.rn.f16x2)", "SHF+IADD (4 pairs)"};
  void (*ks[])(int*, int) = {k_i2f, k_ex2, k_f2h, k_iadd};
  const double ops[] = {4, 4, 2, 8};
  for (int t = 0; t < 4; ++t) {
    ks[t]<<<148 * 8, 1024>>>(o, 16);
    cudaEventRecord(e0);
    ks[t]<<<148 * 8, 1024>>>(o, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double tot = 148.0 * 8 * 1024 * n * ops[t];
    printf("%-28s %.1f ops/clk/SM (at %d MHz)\n", names[t], tot / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
  }
  return 0;
}

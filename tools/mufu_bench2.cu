// Microbenchmark: packed MUFU.EX2 variants (f16x2 / bf16x2) vs f32 on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
template <int MODE>
__global__ void k(uint32_t* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = __float_as_uint(ex2f(__uint_as_float(a[i]) * -0.5f));
      else if (MODE == 1) a[i] = ex2h2(a[i]) ^ 0x80008000u;
      else a[i] = ex2b2(a[i]) ^ 0x80008000u;
    }
  }
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 12345u) out[0] = s;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  const char* names[3] = {"f32", "f16x2", "bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(d, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(d, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double inst = double(blocks) * threads * iters * 8;
      if (rep) printf("%s: %.3f ms, %.2f MUFU-inst/clk/SM (per lane-op), elems/clk/SM %.2f @1965MHz\n", names[mode], ms, inst / (ms * 1e-3) / sms / 1.965e9, inst * (mode ? 2 : 1) / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}

// Microbenchmark: MUFU.EX2 and FMA-pipe throughput per SM on this GPU (informs the softmax design).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) * -0.5f;         // MUFU + FMUL
      else if (MODE == 1) a[i] = fmaf(a[i], 0.999f, 1e-7f);  // FFMA
      else { a[i] = ex2(a[i]) * -0.5f; a[i] = fmaf(a[i], 0.999f, 1e-7f); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(d, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(d, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = double(blocks) * threads * iters * 8;
      if (rep) printf("mode %d: %.3f ms, %.1f Gop/s, %.2f op/clk/SM @ reported max clk %d MHz\n", mode, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}

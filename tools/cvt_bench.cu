// Does cvt.rn.bf16x2.f32 (F2FP) share the MUFU/XU pipe with ex2?  Throughput per SM of: ex2 alone,
// F2FP alone, ex2 + F2FP interleaved (softmax ratio: one pack per two exps), FFMA2-pack mix.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pk(float a, float b) { unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(unsigned* out, int iters) {
  float a[8];
  unsigned acc = 0;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0) { a[i] = ex2(a[i]); a[i + 1] = ex2(a[i + 1]); }
      else if (MODE == 1) { acc ^= pk(a[i], a[i + 1]); a[i] += 1e-7f; }
      else { a[i] = ex2(a[i]); a[i + 1] = ex2(a[i + 1]); acc ^= pk(a[i], a[i + 1]); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f || acc == 0x12345678u) out[0] = acc + unsigned(s);
}
int main() {
  unsigned* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  const char* names[3] = {"ex2 only (per ex2)", "cvt bf16x2 only (per cvt)", "2 ex2 + 1 cvt (per ex2)"};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(d, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(d, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    // clock: measure with clock64 not available here; report ops per ns per SM
    double ops = double(blocks) * threads * iters * (mode == 1 ? 4 : 8);
    printf("%-28s %.3f ms  %.2f op/ns/SM\n", names[mode], best, ops / (best * 1e6) / sms);
  }
  return 0;
}

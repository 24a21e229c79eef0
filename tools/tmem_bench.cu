// Microbenchmark: tcgen05.ld (TMEM -> registers) and tcgen05.st throughput per SM on this GPU.
// One CTA per SM, 4 or 8 warps, each warp repeatedly loads 32 lanes x 32 columns (4 KB) from its
// TMEM lane quarter.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    if (MODE == 2) {
      uint32_t q[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(q[c*32+0]),"=r"(q[c*32+1]),"=r"(q[c*32+2]),"=r"(q[c*32+3]),"=r"(q[c*32+4]),"=r"(q[c*32+5]),"=r"(q[c*32+6]),"=r"(q[c*32+7]),"=r"(q[c*32+8]),"=r"(q[c*32+9]),"=r"(q[c*32+10]),"=r"(q[c*32+11]),"=r"(q[c*32+12]),"=r"(q[c*32+13]),"=r"(q[c*32+14]),"=r"(q[c*32+15]),"=r"(q[c*32+16]),"=r"(q[c*32+17]),"=r"(q[c*32+18]),"=r"(q[c*32+19]),"=r"(q[c*32+20]),"=r"(q[c*32+21]),"=r"(q[c*32+22]),"=r"(q[c*32+23]),"=r"(q[c*32+24]),"=r"(q[c*32+25]),"=r"(q[c*32+26]),"=r"(q[c*32+27]),"=r"(q[c*32+28]),"=r"(q[c*32+29]),"=r"(q[c*32+30]),"=r"(q[c*32+31]) : "r"(tmem + c * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int i = 0; i < 128; ++i) acc ^= q[i];
    } else if (MODE == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(tmem + c * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= r[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = it + i;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
          :: "r"(tmem + c * 32), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(slot), "r"(512));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d; cudaMalloc(&d, sms * 256 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps = 4; warps <= 8; warps += 4)
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<sms, warps * 32>>>(d, iters); else if (mode == 1) k<1><<<sms, warps * 32>>>(d, iters); else k<2><<<sms, warps * 32>>>(d, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = double(sms) * warps * iters * 4 * 32 * 32 * 4;  // per warp: 4 x (32 lanes x 32 cols x 4B)
        if (rep) printf("%s warps=%d: %.3f ms, %.1f B/clk/SM @1.9GHz (%.2f TB/s/SM)  err=%s\n", mode == 1 ? "st" : (mode == 2 ? "ld4-1wait" : "ld"), warps, ms,
                        bytes / (ms * 1e-3) / sms / 1.9e9, bytes / (ms * 1e-3) / sms / 1e12, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}

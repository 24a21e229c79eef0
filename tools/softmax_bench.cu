// Softmax-phase microbenchmark: the forward kernels' per-tile S -> P work (tcgen05.ld of a 128-column
// S row, speculative exp pass with packed FFMA2 / MUFU.EX2 / FADD2 / bf16 pack and tcgen05.st of P)
// run in a loop by 1 or 2 warps per SM sub-partition, one CTA per SM.  Reports cycles per tile per
// warp and the MUFU utilisation this implies (16 ex2/clk/SM).  VARIANT selects the loop form.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/softmax_bench.cu
#include <cstdio>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include "../paper_2604_20819_b200/csrc/ptx.cuh"
using namespace cqs;

__device__ unsigned long long g_cyc[64];
__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <int VARIANT>
__global__ void __launch_bounds__(256, 1) k(int iters, float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tS = slot + (uint32_t((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  {  // fill S with smooth values
    uint32_t v[32];
    for (int c = 0; c < 4; ++c) {
      for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.01f * ((lane * 7 + i * 3 + c) % 50));
      ptx::tmem_st32(tS + c * 32, v);
    }
    ptx::tmem_st_wait();
  }
  const float scale_log2 = 0.1275f;
  float m = 1.0f, l = 0.f, rmax_acc = 0.f;
  __syncwarp();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    uint32_t sr[128];
#pragma unroll
    for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
    ptx::tmem_ld_wait();
    float* s = reinterpret_cast<float*>(sr);
    const uint64_t sc2 = ptx::f2(scale_log2, scale_log2), nm2 = ptx::f2(-m, -m);
    uint64_t rs2[4] = {0, 0, 0, 0};
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int ii = 0; ii < 16; ++ii) {
        const int i = 16 * c + ii;
        if (VARIANT == 3)
          mx4[ii & 3] = max3(mx4[ii & 3], s[2 * i], s[2 * i + 1]);
        else if (VARIANT != 2 && (ii & 1) == 0)
          mx4[(i >> 1) & 3] = fmaxf(mx4[(i >> 1) & 3], fmaxf(fmaxf(s[2 * i], s[2 * i + 1]),
                                                             fmaxf(s[2 * i + 2], s[2 * i + 3])));
        float x0, x1;
        ptx::f2_split(ptx::ffma2(ptx::f2(s[2 * i], s[2 * i + 1]), sc2, nm2), x0, x1);
        x0 = ptx::ex2(x0);
        x1 = ptx::ex2(x1);
        rs2[ii & 3] = ptx::fadd2(rs2[ii & 3], ptx::f2(x0, x1));
        pk[ii] = ptx::pack_bf16(x0, x1);
      }
      if (VARIANT != 1) ptx::tmem_st16(tS + c * 16 + 64, pk);   // P into the upper half (keeps S)
      else rmax_acc += __uint_as_float(pk[0] ^ pk[15]);
    }
    const uint64_t rr = ptx::fadd2(ptx::fadd2(rs2[0], rs2[1]), ptx::fadd2(rs2[2], rs2[3]));
    float a0, a1;
    ptx::f2_split(rr, a0, a1);
    l += a0 + a1;
    rmax_acc += fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
    ptx::tmem_st_wait();
    m += 1e-9f * rmax_acc;   // loop-carried, keeps the max live
  }
  const long long t1 = clock64();
  if (lane == 0) atomicAdd(&g_cyc[0], (unsigned long long)(t1 - t0)), atomicAdd(&g_cyc[1], 1ull);
  if (l == 12345.f) out[0] = l + m;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(slot, 512);
  }
}

template <int V>
void run(const char* name, int warps, float* d) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  unsigned long long z[64] = {};
  cudaMemcpyToSymbol(g_cyc, z, sizeof(z));
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  k<V><<<sms, warps * 32, 150 * 1024>>>(iters, d);   // big smem: one CTA per SM
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[64];
  cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  const double cyc = double(c[0]) / c[1] / iters;   // per tile (128 exps per thread) per warp
  const double per_smsp = warps / 4;                // warps sharing one sub-partition
  // MUFU floor per tile per warp alone: 128 ex2 x 32 lanes / 4 per clk = 1024 cycles; with k warps
  // per sub-partition running concurrently the floor is k x 1024
  printf("%-34s warps/SMSP %d: %7.0f cyc/tile/warp  MUFU util %.2f  (%s)\n", name, int(per_smsp),
         cyc, per_smsp * 1024.0 / cyc, cudaGetErrorString(e));
}

int main() {
  float* d;
  cudaMalloc(&d, 64);
  for (int w : {4, 8}) {
    run<0>("exp pass + max + tcgen05.ld/st", w, d);
    run<1>("exp pass + max, no tcgen05.st", w, d);
    run<3>("exp pass + max3 per pair", w, d);
  }
  return 0;
}

// L2 fp32 reduction throughput: every warp issues coalesced red.global.add.f32 (128 B per warp
// instruction) over a buffer (default 64 MB, like one fp32 dQ accumulator plane set), the access
// pattern of a fused-dQ backward drain.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red_kernel(float* buf, long n, int iters, int vec) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    for (long i = tid; i < n / vec; i += stride) {
      if (vec == 1) {
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(buf + i), "f"(1.0f) : "memory");
      } else {
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(buf + 4 * i), "f"(1.0f),
                     "f"(1.0f), "f"(1.0f), "f"(1.0f)
                     : "memory");
      }
    }
  }
}
int main() {
  for (long mb : {64L, 1024L}) {
    long n = mb * (1 << 20) / 4;
    float* b;
    cudaMalloc(&b, n * 4);
    cudaMemset(b, 0, n * 4);
    for (int vec : {1, 4}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      red_kernel<<<148 * 8, 256>>>(b, n, 1, vec);
      cudaEventRecord(e0);
      int iters = mb == 64 ? 20 : 2;
      red_kernel<<<148 * 8, 256>>>(b, n, iters, vec);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("buffer %ld MB vec%d: %.2f TB/s of fp32 reductions\n", mb, vec,
             double(n) * 4 * iters / (ms * 1e-3) / 1e12);
    }
    cudaFree(b);
  }
  return 0;
}

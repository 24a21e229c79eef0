// Per-task CQS attention kernel, fp32 inputs, CUDA-core FFMA (the 1e-5 parity path, BASELINE
// config 0).  Same task/segment/merge contract as the tcgen05 kernel: the per-task partial of
// Eq. 2 in FA form (O_i, lse_i), merged into the fp32 accumulator in the
// epilogue (Eq. 3).  Online softmax in natural-exp fp32 (expf), one warp per query row at a
// time, lanes over keys for Q.K and over head-dim for P.V.
#include <cuda_runtime.h>

#include "task_params.cuh"

namespace cqs {

constexpr int kF32Rows = 32;     // query rows per CTA (4 warps x 8 rows)
constexpr int kF32Keys = 32;     // keys per tile (one per lane)
constexpr int kF32Threads = 128;

template <int D>
__global__ void __launch_bounds__(kF32Threads)
    attn_f32_kernel(const __grid_constant__ TaskParams tp, const float* __restrict__ q,
                    const float* __restrict__ k, const float* __restrict__ v, int64_t sB,
                    int64_t sH, int64_t sN, float* __restrict__ acc_o,
                    float* __restrict__ acc_lse, float scale) {
  constexpr int NV = D / 32;  // head-dim elements per lane
  constexpr int RPW = kF32Rows / (kF32Threads / 32);
  extern __shared__ float f32_smem[];
  float(*sQ)[D] = reinterpret_cast<float(*)[D]>(f32_smem);                        // [32][D]
  float(*sK)[D + 1] = reinterpret_cast<float(*)[D + 1]>(f32_smem + kF32Rows * D);  // [32][D+1]
  float(*sV)[D] = reinterpret_cast<float(*)[D]>(f32_smem + kF32Rows * D + kF32Keys * (D + 1));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x / tp.n_items, item = blockIdx.x % tp.n_items;  // head-major
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  const int a = tp.order[oi];
  const int q_off = (item - (oi ? tp.item_end[oi - 1] : 0)) * kF32Rows;
  const int vrows = min(kF32Rows, tp.seg_len[a] - q_off);
  const int64_t base = int64_t(bh / tp.H) * sB + int64_t(bh % tp.H) * sH;

  for (int i = threadIdx.x; i < kF32Rows * D; i += kF32Threads) {
    const int r = i / D, d = i % D;
    sQ[r][d] = r < vrows ? q[base + int64_t(tp.seg_src[a] + q_off + r) * sN + d] : 0.f;
  }

  float m[RPW], l[RPW], o[RPW][NV];
#pragma unroll
  for (int rr = 0; rr < RPW; ++rr) {
    m[rr] = -INFINITY;
    l[rr] = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) o[rr][i] = 0.f;
  }

  for (uint32_t msk = tp.kept[a]; msk; msk &= msk - 1) {
    const int b = __ffs(msk) - 1;
    const int len_b = tp.seg_len[b];
    for (int k0 = 0; k0 < len_b; k0 += kF32Keys) {
      const int vk = min(kF32Keys, len_b - k0);
      __syncthreads();
      for (int i = threadIdx.x; i < kF32Keys * D; i += kF32Threads) {
        const int r = i / D, d = i % D;
        const int64_t g = base + int64_t(tp.seg_src[b] + k0 + r) * sN + d;
        sK[r][d] = r < vk ? k[g] : 0.f;
        sV[r][d] = r < vk ? v[g] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int row = warp * RPW + rr;
        float s = 0.f;
#pragma unroll 8
        for (int d = 0; d < D; ++d) s = fmaf(sQ[row][d], sK[lane][d], s);
        s = lane < vk ? s * scale : -INFINITY;
        float mx = s;
#pragma unroll
        for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const float m_new = fmaxf(m[rr], mx);
        const float f = expf(m[rr] - m_new);  // m = -inf on the first tile -> 0
        const float p = expf(s - m_new);
        float ps = p;
#pragma unroll
        for (int off = 16; off; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
        l[rr] = l[rr] * f + ps;
        m[rr] = m_new;
#pragma unroll
        for (int i = 0; i < NV; ++i) o[rr][i] *= f;
        for (int j = 0; j < vk; ++j) {
          const float pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
          for (int i = 0; i < NV; ++i) o[rr][i] = fmaf(pj, sV[j][lane + 32 * i], o[rr][i]);
        }
      }
    }
  }

#pragma unroll
  for (int rr = 0; rr < RPW; ++rr) {
    const int row = warp * RPW + rr;
    if (row >= vrows) continue;
    const float lse = m[rr] + logf(l[rr]);
    const float inv = 1.f / l[rr];
    const int64_t idx = int64_t(tp.seg_dst[a] + q_off + row) * tp.BH + bh;
    const MergeW w = merge_weights(acc_lse[idx], lse);
    float* dst = acc_o + idx * D;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int d = lane + 32 * i;
      const float val = w.wp * (o[rr][i] * inv);
      dst[d] = w.wa != 0.f ? fmaf(w.wa, dst[d], val) : val;
    }
    __syncwarp();
    if (lane == 0) acc_lse[idx] = w.lse;
  }
}

template <int D>
static cudaError_t launch_f32_impl(int64_t grid, const TaskParams& tp, const float* q,
                                   const float* k, const float* v, const int64_t* strides,
                                   float* acc_o, float* acc_lse, float scale, cudaStream_t stream) {
  constexpr int smem = (kF32Rows * D + kF32Keys * (D + 1) + kF32Keys * D) * 4;
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = set_smem_attr_once(attn_f32_kernel<D>, smem, configured);
  if (e != cudaSuccess) return e;
  attn_f32_kernel<D><<<dim3(unsigned(grid)), kF32Threads, smem, stream>>>(
      tp, q, k, v, strides[0], strides[1], strides[2], acc_o, acc_lse, scale);
  return cudaGetLastError();
}

cudaError_t launch_attn_f32(int D, const TaskParams& tp, const float* q, const float* k,
                            const float* v, const int64_t* strides, float* acc_o, float* acc_lse,
                            float scale, cudaStream_t stream) {
  const int64_t grid = int64_t(tp.n_items) * tp.BH;
  if (grid <= 0) return cudaSuccess;
  switch (D) {
    case 32: return launch_f32_impl<32>(grid, tp, q, k, v, strides, acc_o, acc_lse, scale, stream);
    case 64: return launch_f32_impl<64>(grid, tp, q, k, v, strides, acc_o, acc_lse, scale, stream);
    case 96: return launch_f32_impl<96>(grid, tp, q, k, v, strides, acc_o, acc_lse, scale, stream);
    case 128: return launch_f32_impl<128>(grid, tp, q, k, v, strides, acc_o, acc_lse, scale, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cqs

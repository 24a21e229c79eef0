// Per-task launch descriptor shared by the attention kernels (passed by value as a kernel param),
// and the fused LSE-merge epilogue helpers.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/cqs.h"

namespace cqs {

// One CQS task (leaf subsequence) as the kernels see it.  A work item is one tile of query rows
// of one active query segment for one (b,h) plane; it loops over the key tiles of every key
// segment its segment keeps (segment-pair block skipping).
struct TaskParams {
  int32_t nseg;
  int32_t n_active;                 // query segments with at least one kept key segment
  int32_t n_items;                  // work items per (b,h) plane
  int32_t BH, H;
  int32_t seg_src[CQS_MAX_SEGS];    // first row of the segment in Q/K/V (TMA / pointer) coords
  int32_t seg_dst[CQS_MAX_SEGS];    // first row of the segment in the fp32 accumulator
  int32_t seg_len[CQS_MAX_SEGS];
  uint32_t kept[CQS_MAX_SEGS];      // bit b: query segment a keeps key segment b
  int32_t order[CQS_MAX_SEGS];      // active query segments, heaviest key work first
  int32_t item_end[CQS_MAX_SEGS];   // cumulative work items after order[i]
};

// Eq. 3 in LSE form: weights to merge a row partial (lse_p) into an accumulator
// row (lse_a).  -inf means "no contribution" (R8); the accumulator's O is ignored when lse_a=-inf.
struct MergeW {
  float wa, wp, lse;
};
__device__ __forceinline__ MergeW merge_weights(float la, float lp) {
  MergeW w;
  if (la == -INFINITY) {
    w.wa = 0.f, w.wp = 1.f, w.lse = lp;
  } else if (lp == -INFINITY) {
    w.wa = 1.f, w.wp = 0.f, w.lse = la;
  } else {
    const float mx = fmaxf(la, lp);
    const float ea = expf(la - mx), ep = expf(lp - mx), s = ea + ep;
    w.wa = ea / s, w.wp = ep / s, w.lse = mx + logf(s);
  }
  return w;
}
// acc[0..NV) = wa * acc + wp * o   (acc 16-byte aligned; never reads acc when wa == 0)
template <int NV>
__device__ __forceinline__ void merge_chunk(float* __restrict__ acc, const float* o, MergeW w) {
  float4* dst = reinterpret_cast<float4*>(acc);
#pragma unroll
  for (int i = 0; i < NV / 4; ++i) {
    float4 r = make_float4(w.wp * o[4 * i + 0], w.wp * o[4 * i + 1], w.wp * o[4 * i + 2],
                           w.wp * o[4 * i + 3]);
    if (w.wa != 0.f) {
      const float4 a = dst[i];
      r.x = fmaf(w.wa, a.x, r.x);
      r.y = fmaf(w.wa, a.y, r.y);
      r.z = fmaf(w.wa, a.z, r.z);
      r.w = fmaf(w.wa, a.w, r.w);
    }
    dst[i] = r;
  }
}

// Dynamic-smem opt-in is a per-device function attribute: set it once per (kernel, device).
template <class Kernel>
inline cudaError_t set_smem_attr_once(Kernel kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

}  // namespace cqs

// Shared pieces of the per-task attention kernels.
#pragma once
#include "task_params.cuh"

namespace cqs {

constexpr int kBM = 128;   // query rows per tile (TMEM lanes)
constexpr int kBN = 128;   // keys per KV tile

// Iterates the key tiles of the kept key segments of one query segment (ascending segment id).
struct KvCursor {
  uint32_t mask;
  int seg, kt, ntile;
  const TaskParams* tp;
  __device__ __forceinline__ void set_seg() {
    seg = mask ? __ffs(mask) - 1 : 0;
    kt = 0;
    ntile = mask ? (tp->seg_len[seg] + kBN - 1) / kBN : 0;
  }
  __device__ __forceinline__ void init(const TaskParams* p, uint32_t m) {
    tp = p;
    mask = m;
    set_seg();
  }
  __device__ __forceinline__ int row() const { return tp->seg_src[seg] + kt * kBN; }
  __device__ __forceinline__ int valid() const { return min(kBN, tp->seg_len[seg] - kt * kBN); }
  __device__ __forceinline__ void next() {
    if (++kt == ntile) {
      mask &= mask - 1;
      set_seg();
    }
  }
};

}  // namespace cqs

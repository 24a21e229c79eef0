// Shared pieces of the per-task attention kernels.
#pragma once
#include "task_params.cuh"

namespace cqs {

constexpr int kBM = 128;   // query rows per tile (TMEM lanes)
constexpr int kBN = 128;   // keys per KV tile

// Iterates the key tiles of the kept key segments of one query segment (ascending segment id),
// starting at tile `start` of that sequence and wrapping around, so exactly n_kv calls of next()
// visit every tile once.  Work items start at different tiles (kv_start below) so the CTAs in
// flight do not all request the same K/V lines from L2 at the same moment; the softmax is
// order-independent (online max / LSE), only the fp32 rounding order changes.
template <int BN = kBN>
struct KvCursorT {
  uint32_t mask0, mask;
  int seg, kt, ntile;
  const TaskParams* tp;
  __device__ __forceinline__ void set_seg() {
    seg = mask ? __ffs(mask) - 1 : 0;
    kt = 0;
    ntile = mask ? (tp->seg_len[seg] + BN - 1) / BN : 0;
  }
  __device__ __forceinline__ void init(const TaskParams* p, uint32_t m, int start = 0) {
    tp = p;
    mask0 = mask = m;
    set_seg();
    while (mask && start >= ntile) {
      start -= ntile;
      mask &= mask - 1;
      set_seg();
    }
    kt = start;
  }
  __device__ __forceinline__ int row() const { return tp->seg_src[seg] + kt * BN; }
  __device__ __forceinline__ int valid() const { return min(BN, tp->seg_len[seg] - kt * BN); }
  __device__ __forceinline__ void next() {
    if (++kt == ntile) {
      mask &= mask - 1;
      if (!mask) mask = mask0;
      set_seg();
    }
  }
};
using KvCursor = KvCursorT<kBN>;

// First KV tile of work item `item` (of n_kv tiles).  CQS_KV_STAGGER = tile stride between
// consecutive items (0: every item starts at tile 0).
#ifndef CQS_KV_STAGGER
#define CQS_KV_STAGGER 0
#endif
__device__ __forceinline__ int kv_start(int item, int n_kv) {
  return CQS_KV_STAGGER == 0 || n_kv == 0 ? 0 : int((uint32_t(item) * CQS_KV_STAGGER) % uint32_t(n_kv));
}

}  // namespace cqs

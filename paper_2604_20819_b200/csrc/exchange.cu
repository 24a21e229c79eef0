// The multi-GPU exchange step (PAPER.md P:136 tasks "distributed across multiple
// devices", "inter-device communication can be entirely avoided" during compute).
//
// With world > 1 every rank runs its tasks into a rank-local fp32 accumulator that holds only the
// rows its tasks touch (blocks of CQS_ACC_BLOCK_ROWS rows, packed in increasing global order; see
// cqs_partial_runs).  The owner of each contiguous row shard then merges, per row, the partials of
// the ranks that hold it (Eq. 3 in LSE form, P:48-52 with Den = exp(lse)) and writes the
// final O / lse: cqs_exchange_merge launches one merge kernel (merge.cu) per maximal run of rows
// held by the same set of ranks, reading the partials over peer memory (NVLink / NVSwitch) or from
// all-to-all receive buffers.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "cqs_internal.h"

namespace cqs {
cudaError_t launch_merge(int64_t rows, int B, int H, int D, int n_parts, const float* const* po,
                         const float* const* pl, float* acc_o, float* acc_lse, bool acc_write,
                         void* out, cqs_dtype out_dtype, const int64_t* out_strides,
                         int64_t out_row0, int64_t n_total, float* lse_out, cudaStream_t st);

// Held blocks -> local block index of rank r (-1 = not held).  World = 1: identity.
static std::vector<int32_t> slots_of(const cqs_plan_t* p, int32_t r) {
  std::vector<uint8_t> held;
  held_blocks(p->tasks, p->segs, p->desc.N, r, held);
  std::vector<int32_t> slot(held.size(), -1);
  int32_t nb = 0;
  for (size_t b = 0; b < held.size(); ++b)
    if (held[b]) slot[b] = nb++;
  return slot;
}

// Runs (global_start, len, local_row) of rank r's accumulator inside [row0, row0 + rows).
static void runs_of(const cqs_plan_t* p, int32_t r, int64_t row0, int64_t rows,
                    std::vector<int64_t>& out) {
  out.clear();
  if (p->desc.world == 1) {
    if (rows > 0) out.insert(out.end(), {row0, rows, row0});
    return;
  }
  const std::vector<int32_t> slot = slots_of(p, r);
  const int64_t G = CQS_ACC_BLOCK_ROWS;
  int64_t g = row0;
  const int64_t end = row0 + rows;
  while (g < end) {
    const int64_t b = g / G, bend = std::min(end, (b + 1) * G);
    if (slot[size_t(b)] >= 0) {
      const int64_t local = int64_t(slot[size_t(b)]) * G + g % G;
      const size_t n = out.size();
      if (n >= 3 && out[n - 3] + out[n - 2] == g && out[n - 1] + out[n - 2] == local)
        out[n - 2] += bend - g;
      else
        out.insert(out.end(), {g, bend - g, local});
    }
    g = bend;
  }
}

}  // namespace cqs

using namespace cqs;

extern "C" cqs_status cqs_partial_runs(const cqs_plan_t* p, int32_t src_rank, int64_t row0,
                                       int64_t rows, int64_t* runs, int64_t max_runs,
                                       int64_t* n_runs) {
  if (!p || !n_runs) return fail(CQS_E_INVALID, "NULL argument");
  if (src_rank < 0 || src_rank >= p->desc.world) return fail(CQS_E_INVALID, "bad src_rank");
  if (row0 < 0 || rows < 0 || row0 + rows > p->desc.N) return fail(CQS_E_INVALID, "bad row range");
  std::vector<int64_t> v;
  runs_of(p, src_rank, row0, rows, v);
  *n_runs = int64_t(v.size() / 3);
  if (!runs) return CQS_OK;
  if (max_runs < *n_runs) return fail(CQS_E_INVALID, "runs buffer too small");
  std::copy(v.begin(), v.end(), runs);
  return CQS_OK;
}

extern "C" cqs_status cqs_exchange_merge(const cqs_plan_t* p, const float* const* part_o,
                                         const float* const* part_lse, const int64_t* part_row0,
                                         void* out, const int64_t out_strides[4], float* lse_out,
                                         void* stream) {
  if (!p || !part_o || !part_lse || !part_row0 || !out || !out_strides)
    return fail(CQS_E_INVALID, "NULL argument");
  const cqs_plan_desc& d = p->desc;
  const int W = d.world;
  if (W < 2) return fail(CQS_E_INVALID, "cqs_exchange_merge needs a world > 1 plan");
  if (W > 16) return fail(CQS_E_UNSUPPORTED, "at most 16 ranks per merge");
  if (out_strides[3] != 1) return fail(CQS_E_INVALID, "out strides: stride(D) must be 1");
  const int64_t row0 = (d.N * d.rank) / W, rows = p->shard_rows;
  const int64_t BH = int64_t(d.B) * d.H, D = d.D;
  // per rank: its runs inside my shard; elementary intervals over all run boundaries
  std::vector<std::vector<int64_t>> rr(static_cast<size_t>(W));
  std::vector<int64_t> cuts{row0, row0 + rows};
  for (int r = 0; r < W; ++r) {
    if (!part_o[r] || !part_lse[r]) return fail(CQS_E_INVALID, "NULL part pointer");
    runs_of(p, r, row0, rows, rr[size_t(r)]);
    for (size_t i = 0; i < rr[size_t(r)].size(); i += 3) {
      cuts.push_back(rr[size_t(r)][i]);
      cuts.push_back(rr[size_t(r)][i] + rr[size_t(r)][i + 1]);
    }
  }
  std::sort(cuts.begin(), cuts.end());
  cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
  std::vector<size_t> at(static_cast<size_t>(W), 0);   // current run of each rank
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (size_t c = 0; c + 1 < cuts.size(); ++c) {
    const int64_t g0 = cuts[c], n = cuts[c + 1] - g0;
    if (g0 < row0 || g0 >= row0 + rows || n <= 0) continue;
    const float* po[16];
    const float* pl[16];
    int np = 0;
    for (int r = 0; r < W; ++r) {
      const std::vector<int64_t>& v = rr[size_t(r)];
      size_t& i = at[size_t(r)];
      while (i < v.size() && v[i] + v[i + 1] <= g0) i += 3;
      if (i < v.size() && v[i] <= g0) {   // rank r holds [g0, g0 + n)
        const int64_t x = v[i + 2] + (g0 - v[i]) - part_row0[r];
        po[np] = part_o[r] + x * BH * D;
        pl[np] = part_lse[r] + x * BH;
        ++np;
      }
    }
    if (np == 0) return fail(CQS_E_VERIFY, "row " + std::to_string(g0) + " is held by no rank");
    cudaError_t e = launch_merge(n, d.B, d.H, d.D, np, po, pl, nullptr, nullptr, false, out,
                                 d.out_dtype, out_strides, g0 - row0, rows, lse_out, st);
    if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("exchange merge: ") + cudaGetErrorString(e));
  }
  return CQS_OK;
}

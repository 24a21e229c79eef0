// Internal declarations shared by the libcqs translation units (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/cqs.h"

namespace cqs {

// Thread-local error message (cqs_last_error).
cqs_status fail(cqs_status st, const std::string& msg);

struct Seg {
  int64_t start;                 // global token id of the first token
  int64_t len;
  uint8_t codes[CQS_MAX_DEPTH];  // per level: index of its chunk in I order (0 = owner)
};

struct Task {
  int32_t nseg = 0;
  int32_t rank = -1;
  int32_t depth = 0;             // leaf depth (uniform plans: the plan depth; hybrid: per leaf)
  uint64_t work = 0;
  int64_t seg_off = 0;           // into cqs_plan::segs
  int32_t quorum[CQS_MAX_DEPTH] = {};
  uint32_t kept[CQS_MAX_SEGS] = {};
};

// Interest sets per divide level ("different values of c ... at each iteration"): level t
// uses (lc[t], lI[t]) for t < lc.size(), the base (c, I) below that.
struct Levels {
  int32_t c = 7;
  std::vector<int32_t> I;
  std::vector<int32_t> lc;
  std::vector<std::vector<int32_t>> lI;
  int c_at(int t) const { return t < int(lc.size()) ? lc[size_t(t)] : c; }
  const std::vector<int32_t>& I_at(int t) const { return t < int(lc.size()) ? lI[size_t(t)] : I; }
  bool mixed() const { return !lc.empty(); }
  int64_t tasks(int depth) const {   // number of leaves of the uniform depth-`depth` tree
    int64_t n = 1;
    for (int t = 0; t < depth; ++t) n *= c_at(t);
    return n;
  }
};

}  // namespace cqs

struct cqs_plan_s {
  cqs_plan_desc desc;                // offsets / level pointers re-pointed at lv below
  cqs::Levels lv;
  std::vector<int32_t> level_offsets;  // concatenated lv.lI (desc.level_offsets points here)
  int32_t depth = 0;                 // base (uniform) depth; hybrid leaves are at depth >= this
  int32_t max_depth = 0;             // deepest leaf
  int32_t acc_depth = 0;             // streamed mode accumulator tier
  int32_t n_stage_buffers = 0;
  std::vector<cqs::Task> tasks;      // c^depth, lexicographic
  std::vector<cqs::Seg> segs;        // CSR storage of task segments
  std::vector<int64_t> my_order;     // non-empty tasks of `rank`, execution order
  // world > 1: rank-local accumulator = the blocks of CQS_ACC_BLOCK_ROWS rows holding a query row
  // of this rank's tasks, packed in increasing global order; acc_slot[block] = local block or -1.
  // Empty when world = 1 (identity over N rows).
  std::vector<int32_t> acc_slot;
  int64_t shard_rows = 0;            // world > 1: rows of this rank's output shard
  int64_t n_empty = 0, max_task_rows = 0, max_staged_rows = 0, max_acc_rows = 0;
  // accumulator row of global row g (segments never straddle an unheld block: all rows of an
  // active query segment are held, so a segment's accumulator rows are consecutive)
  int64_t acc_row(int64_t g) const {
    if (acc_slot.empty()) return g;
    const int32_t s = acc_slot[size_t(g / CQS_ACC_BLOCK_ROWS)];
    return s < 0 ? -1 : int64_t(s) * CQS_ACC_BLOCK_ROWS + g % CQS_ACC_BLOCK_ROWS;
  }
  uint64_t total_work = 0, my_work = 0;
  uint64_t dev_ws = 0, host_ws = 0, predicted_peak = 0;
};

namespace cqs {
// Memory model (plan.cpp).  acc_rows = rows of the device accumulator tier.
struct MemModel {
  uint64_t caller_dev, dev_ws, host_ws;
};
// out_rows: rows of O / lse the call's caller holds on the device (N; world > 1: the output shard,
// which the exchange writes on the device whatever out_loc says).
MemModel memory_model(const cqs_plan_desc& d, int64_t staged_rows, int64_t acc_rows,
                      int32_t n_stage_buffers, int64_t out_rows);
// Held accumulator blocks (CQS_ACC_BLOCK_ROWS rows) of rank r under the current Task::rank values.
void held_blocks(const std::vector<Task>& tasks, const std::vector<Seg>& segs, int64_t N,
                 int32_t r, std::vector<uint8_t>& held);
uint64_t align256(uint64_t x);
uint64_t alloc_bytes(uint64_t x);
// Section offsets of the device workspace (forward.cu must follow memory_model exactly).
struct WsLayout {
  uint64_t acc_o, acc_lse, stage, stage_bytes_per_buf, flush, slots, slot_bytes, total;
};
WsLayout ws_layout(const cqs_plan_desc& d, int64_t staged_rows, int64_t acc_rows,
                   int32_t n_stage_buffers);
// Flush buffers (streamed mode): two buffers of F rows x B*H x (D+1) fp32 with
// F = clamp(kFlushBytes / (B*H*(D+1)*4), 1024, 65536), never more than the accumulator rows.
constexpr int64_t kFlushBytes = 256ll << 20;
inline int64_t flush_rows(int64_t acc_rows, int64_t BH, int64_t D) {
  int64_t f = kFlushBytes / (BH * (D + 1) * 4);
  f = f < 1024 ? 1024 : (f > 65536 ? 65536 : f);
  return f < acc_rows ? f : acc_rows;
}
// Segments of the depth-`depth` subsequence selected by quorum[0..depth) (Alg. 3).
bool build_segments(int64_t N, const Levels& lv, const int32_t* quorum, int depth,
                    std::vector<Seg>& out);
}  // namespace cqs

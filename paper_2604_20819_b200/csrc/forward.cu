// Forward executor (Algorithm 1 in LSE form): for every task of this
// rank, in plan order, launch the per-task attention kernel whose epilogue LSE-merges the task's
// partial into the fp32 accumulator (IndexAdd of P:72-73), then finalize O / lse.
//
// Resident mode: Q/K/V stay in the caller's HBM tensors; the kernels address each task's
// segments directly through TMA tensor maps (Gather of P:66 without a copy).
// Streamed mode (Q/K/V in pinned host memory): see stream.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "cqs_internal.h"
#include "task_params.cuh"

namespace cqs {

cudaError_t launch_attn_bf16(int D, const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                             float* acc_lse, float scale, cudaStream_t stream);
cudaError_t launch_attn_f32(int D, const TaskParams& tp, const float* q, const float* k,
                            const float* v, const int64_t* strides, float* acc_o, float* acc_lse,
                            float scale, cudaStream_t stream);
cudaError_t launch_fill(float* p, int64_t n, float val, cudaStream_t st);
int attn_rows_per_item(int D);
int attn_box_rows(int D, int which);
cudaError_t launch_merge(int64_t rows, int B, int H, int D, int n_parts, const float* const* po,
                         const float* const* pl, float* acc_o, float* acc_lse, bool acc_write,
                         void* out, cqs_dtype out_dtype, const int64_t* out_strides,
                         int64_t out_row0, int64_t n_total, float* lse_out, cudaStream_t st);

// ---- TMA tensor maps (driver entry point fetched through the runtime; no -lcuda needed) ----
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [B][H][rows][D] bf16 with element strides (sB, sH, sN, 1); box = 64 columns x box_rows rows.
cqs_status make_tmap_bf16(CUtensorMap* m, const void* base, int B, int H, int64_t rows, int D,
                          int64_t sB, int64_t sH, int64_t sN, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(CQS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (sN * 2) % 16 || (sH * 2) % 16 || (sB * 2) % 16)
    return fail(CQS_E_INVALID, "TMA needs 16-byte aligned base and row/plane strides");
  cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(rows), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(sN * 2), cuuint64_t(std::max<int64_t>(sH, 8) * 2),
                           cuuint64_t(std::max<int64_t>(sB, 8) * 2)};
  cuuint32_t box[4] = {64, cuuint32_t(box_rows), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(CQS_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return CQS_OK;
}

// Build the kernel descriptor of task T.  src_of(a) gives a segment's first row in the Q/K/V
// coordinate space, dst_of(a) its first accumulator row.
template <class Src, class Dst>
static void build_task_params(const cqs_plan_t* p, const Task& T, int rows_per_item, Src src_of,
                              Dst dst_of, TaskParams& tp) {
  std::memset(&tp, 0, sizeof(tp));
  tp.nseg = T.nseg;
  tp.BH = p->desc.B * p->desc.H;
  tp.H = p->desc.H;
  int64_t keywork[CQS_MAX_SEGS] = {};
  int act[CQS_MAX_SEGS], na = 0;
  for (int a = 0; a < T.nseg; ++a) {
    const Seg& s = p->segs[size_t(T.seg_off + a)];
    tp.seg_src[a] = int32_t(src_of(a));
    tp.seg_dst[a] = int32_t(dst_of(a));
    tp.seg_len[a] = int32_t(s.len);
    tp.kept[a] = T.kept[a];
    for (int b = 0; b < T.nseg; ++b)
      if (T.kept[a] >> b & 1) keywork[a] += p->segs[size_t(T.seg_off + b)].len;
    if (T.kept[a]) act[na++] = a;
  }
  // heaviest key work first (LPT inside the launch); ties keep segment order
  std::stable_sort(act, act + na, [&](int x, int y) { return keywork[x] > keywork[y]; });
  int items = 0;
  for (int i = 0; i < na; ++i) {
    tp.order[i] = act[i];
    items += int((tp.seg_len[act[i]] + rows_per_item - 1) / rows_per_item);
    tp.item_end[i] = items;
  }
  for (int i = na; i < CQS_MAX_SEGS; ++i) tp.item_end[i] = items + 1;  // never reached
  tp.n_active = na;
  tp.n_items = items;
}

void build_task_params_ext(const cqs_plan_t* p, const Task& T, int rows_per_item,
                           const int64_t* src_rows, const int64_t* dst_rows, TaskParams& tp) {
  build_task_params(
      p, T, rows_per_item, [&](int a) { return src_rows[a]; }, [&](int a) { return dst_rows[a]; },
      tp);
}

// Descriptor of an explicit segment list (the streamed executor's first task split into pieces):
// nseg segments of len[a] rows, kept[a] over those segments.
void build_task_params_raw(int BH, int H, int nseg, const int64_t* len, const uint32_t* kept,
                           int rows_per_item, const int64_t* src_rows, const int64_t* dst_rows,
                           TaskParams& tp) {
  std::memset(&tp, 0, sizeof(tp));
  tp.nseg = nseg;
  tp.BH = BH;
  tp.H = H;
  int64_t keywork[CQS_MAX_SEGS] = {};
  int act[CQS_MAX_SEGS], na = 0;
  for (int a = 0; a < nseg; ++a) {
    tp.seg_src[a] = int32_t(src_rows[a]);
    tp.seg_dst[a] = int32_t(dst_rows[a]);
    tp.seg_len[a] = int32_t(len[a]);
    tp.kept[a] = kept[a];
    for (int b = 0; b < nseg; ++b)
      if (kept[a] >> b & 1) keywork[a] += len[b];
    if (kept[a]) act[na++] = a;
  }
  std::stable_sort(act, act + na, [&](int x, int y) { return keywork[x] > keywork[y]; });
  int items = 0;
  for (int i = 0; i < na; ++i) {
    tp.order[i] = act[i];
    items += int((tp.seg_len[act[i]] + rows_per_item - 1) / rows_per_item);
    tp.item_end[i] = items;
  }
  for (int i = na; i < CQS_MAX_SEGS; ++i) tp.item_end[i] = items + 1;
  tp.n_active = na;
  tp.n_items = items;
}

cqs_status forward_streamed(const cqs_plan_t* p, const void* q, const void* k, const void* v,
                            void* out, const int64_t* out_strides, float* lse, float scale,
                            uint8_t* ws, uint8_t* host_ws, cudaStream_t st, cqs_stats* stats);

}  // namespace cqs

using namespace cqs;

extern "C" cqs_status cqs_partial_view(const cqs_plan_t* p, void* dev_ws, float** acc_o,
                                       float** acc_lse) {
  if (!p || !dev_ws || !acc_o || !acc_lse) return fail(CQS_E_INVALID, "NULL argument");
  if (p->desc.world == 1 && p->desc.qkv_loc != CQS_LOC_DEVICE)
    return fail(CQS_E_UNSUPPORTED, "partial view: resident or world > 1 plans only");
  const WsLayout L = ws_layout(p->desc, p->max_staged_rows, p->max_acc_rows, p->n_stage_buffers);
  *acc_o = reinterpret_cast<float*>(static_cast<uint8_t*>(dev_ws) + L.acc_o);
  *acc_lse = reinterpret_cast<float*>(static_cast<uint8_t*>(dev_ws) + L.acc_lse);
  return CQS_OK;
}

extern "C" cqs_status cqs_attention_forward(const cqs_plan_t* p, const void* q, const void* k,
                                            const void* v, const int64_t qkv_strides[4],
                                            void* out, const int64_t out_strides[4], float* lse,
                                            float scale, uint64_t budget_bytes, void* dev_ws,
                                            void* host_ws, void* stream_, cqs_stats* stats) {
  if (!p) return fail(CQS_E_INVALID, "plan is NULL");
  const cqs_plan_desc& d = p->desc;
  if (!q || !k || !v) return fail(CQS_E_INVALID, "q/k/v NULL");
  if (d.world == 1 && !out) return fail(CQS_E_INVALID, "out NULL");
  if (!dev_ws && p->dev_ws) return fail(CQS_E_OOM, "device workspace missing");
  if (!host_ws && p->host_ws) return fail(CQS_E_OOM, "pinned host workspace missing");
  if (reinterpret_cast<uintptr_t>(dev_ws) & 255) return fail(CQS_E_INVALID, "dev_ws must be 256B aligned");
  if (budget_bytes && p->predicted_peak > budget_bytes)
    return fail(CQS_E_INFEASIBLE, "plan's predicted peak exceeds budget_bytes");
  if (out && (!out_strides || out_strides[3] != 1))
    return fail(CQS_E_INVALID, "out strides: stride(D) must be 1");
  if (scale <= 0.f) scale = 1.f / std::sqrt(float(d.D));
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  const auto t0 = std::chrono::steady_clock::now();
  uint8_t* ws = static_cast<uint8_t*>(dev_ws);

  if (d.qkv_loc == CQS_LOC_PINNED_HOST) {
    // the staging copies address rows as base + row * D with pitch N * D: contiguous only
    const int64_t N = d.N, D = d.D;
    if (!qkv_strides || qkv_strides[0] != int64_t(d.H) * N * D || qkv_strides[1] != N * D ||
        qkv_strides[2] != D || qkv_strides[3] != 1)
      return fail(CQS_E_INVALID, "streamed Q/K/V must be contiguous [B,H,N,D]");
    return forward_streamed(p, q, k, v, out, out_strides, lse, scale, ws,
                            static_cast<uint8_t*>(host_ws), st, stats);
  }

  if (!qkv_strides || qkv_strides[3] != 1)
    return fail(CQS_E_INVALID, "qkv strides: stride(D) must be 1");
  const int BH = d.B * d.H;
  const WsLayout L = ws_layout(d, 0, p->max_acc_rows, 0);
  // n_parallel > 1: slot s in [0, P) = stream s (0 = the caller's) + its own accumulator
  const int P = std::max(1, int(d.n_parallel));
  std::vector<float*> slot_o(static_cast<size_t>(P)), slot_l(static_cast<size_t>(P));
  for (int s = 0; s < P; ++s) {
    uint8_t* base = s == 0 ? ws : ws + L.slots + uint64_t(s - 1) * L.slot_bytes;
    slot_o[size_t(s)] = reinterpret_cast<float*>(base + (s == 0 ? L.acc_o : 0));
    slot_l[size_t(s)] = reinterpret_cast<float*>(
        base + (s == 0 ? L.acc_lse : align256(uint64_t(p->max_acc_rows) * BH * d.D * 4)));
  }
  float* acc_o = slot_o[0];
  float* acc_lse = slot_l[0];
  int64_t launches = 0;
  // stats: CUDA events around every launch on `st` (kernel durations, not host time); with P > 1
  // one pair around all tasks (they overlap across streams)
  std::vector<cudaEvent_t> evs;
  auto mark = [&]() {
    if (!stats) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, st);
    evs.push_back(ev);
  };
  mark();
  cudaError_t e = cudaSuccess;
  for (int s = 0; s < P && e == cudaSuccess; ++s, ++launches)
    e = launch_fill(slot_l[size_t(s)], p->max_acc_rows * BH, -INFINITY, st);
  mark();
  if (e != cudaSuccess) return fail(CQS_E_CUDA, cudaGetErrorString(e));
  struct Streams {   // helper streams + events of the P > 1 mode, released on every return path
    std::vector<cudaStream_t> s;
    std::vector<cudaEvent_t> e;
    ~Streams() {
      for (auto x : e) cudaEventDestroy(x);
      for (auto x : s) cudaStreamDestroy(x);
    }
  } ps;
  std::vector<cudaStream_t> sts(size_t(P), st);
  if (P > 1) {
    cudaEvent_t filled;
    if ((e = cudaEventCreateWithFlags(&filled, cudaEventDisableTiming)) != cudaSuccess)
      return fail(CQS_E_CUDA, cudaGetErrorString(e));
    ps.e.push_back(filled);
    cudaEventRecord(filled, st);
    for (int s = 1; s < P; ++s) {
      cudaStream_t x;
      if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(CQS_E_CUDA, cudaGetErrorString(e));
      ps.s.push_back(x);
      sts[size_t(s)] = x;
      cudaStreamWaitEvent(x, filled, 0);
    }
  }

  CUtensorMap maps[3];
  if (d.in_dtype == CQS_BF16) {
    const void* bases[3] = {q, k, v};
    for (int i = 0; i < 3; ++i) {
      cqs_status s = make_tmap_bf16(&maps[i], bases[i], d.B, d.H, d.N, d.D, qkv_strides[0],
                                    qkv_strides[1], qkv_strides[2],
                                    attn_box_rows(d.D, i));
      if (s != CQS_OK) return s;
    }
  }
  const int rows_per_item = d.in_dtype == CQS_BF16 ? attn_rows_per_item(d.D) : 32;
  TaskParams tp;
  int64_t run = 0;
  for (int64_t ti : p->my_order) {
    const Task& T = p->tasks[size_t(ti)];
    const int slot = int(run % P);
    auto seg_start = [&](int a) { return p->segs[size_t(T.seg_off + a)].start; };
    auto seg_acc = [&](int a) { return p->acc_row(p->segs[size_t(T.seg_off + a)].start); };
    build_task_params(p, T, rows_per_item, seg_start, seg_acc, tp);
    if (P == 1) mark();
    cudaStream_t ts = sts[size_t(slot)];
    if (d.in_dtype == CQS_BF16)
      e = launch_attn_bf16(d.D, maps, tp, slot_o[size_t(slot)], slot_l[size_t(slot)], scale, ts);
    else
      e = launch_attn_f32(d.D, tp, static_cast<const float*>(q), static_cast<const float*>(k),
                          static_cast<const float*>(v), qkv_strides, slot_o[size_t(slot)],
                          slot_l[size_t(slot)], scale, ts);
    if (P == 1) mark();
    if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
    ++launches;
    ++run;
  }
  if (P > 1) {   // join the helper streams, then fold slots 1..P-1 into slot 0 (Eq. 3)
    for (int s = 1; s < P; ++s) {
      cudaEvent_t done;
      if ((e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming)) != cudaSuccess)
        return fail(CQS_E_CUDA, cudaGetErrorString(e));
      ps.e.push_back(done);
      cudaEventRecord(done, sts[size_t(s)]);
      cudaStreamWaitEvent(st, done, 0);
    }
    mark();
    if (d.world > 1) {   // the exchange reads slot 0: merge the others into it in place
      e = launch_merge(p->max_acc_rows, d.B, d.H, d.D, P - 1, slot_o.data() + 1,
                       slot_l.data() + 1, acc_o, acc_lse, true, nullptr, d.out_dtype, nullptr, 0,
                       p->max_acc_rows, nullptr, st);
      ++launches;
      if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("slot merge: ") + cudaGetErrorString(e));
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (d.world == 1) {
    if (P == 1) mark();
    // finalize (P > 1: the slots' merge and the finalize in one kernel)
    e = launch_merge(d.N, d.B, d.H, d.D, P - 1, P > 1 ? slot_o.data() + 1 : nullptr,
                     P > 1 ? slot_l.data() + 1 : nullptr, acc_o, acc_lse, false, out,
                     d.out_dtype, out_strides, 0, d.N, lse, st);
    mark();
    ++launches;
    if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("finalize: ") + cudaGetErrorString(e));
  } else if (P > 1) {
    mark();
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(CQS_E_CUDA, cudaGetErrorString(e));
    const auto t2 = std::chrono::steady_clock::now();
    stats->ms_total = std::chrono::duration<double, std::milli>(t2 - t0).count();
    (void)t1;
    // P = 1 pairs: [fill] [task_0] ... [task_{run-1}] [finalize];  P > 1: [fill] [all tasks]
    // [merge + finalize]
    const size_t n_attn = P == 1 ? size_t(run) : 1;
    for (size_t i = 0; i + 1 < evs.size(); i += 2) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, evs[i], evs[i + 1]);
      const bool is_attn = i >= 2 && i < 2 + 2 * n_attn;
      (is_attn ? stats->ms_attn : stats->ms_merge) += ms;
    }
    for (auto ev : evs) cudaEventDestroy(ev);
    stats->tasks_run = run;
    stats->tasks_skipped = int64_t(p->tasks.size()) - run;
    stats->kernel_launches = launches;
    stats->predicted_peak_bytes = p->predicted_peak;
  }
  return CQS_OK;
}

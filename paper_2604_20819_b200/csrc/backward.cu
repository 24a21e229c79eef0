// Backward executor (Algorithm 2): Delta / lse prep, then for every task of the
// plan the dK/dV and dQ kernels (attn_bwd_sm100.cu) that IndexAdd the task's gradients into fp32
// accumulators, then a cast of the accumulators into the caller's dQ/dK/dV.
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "cqs_internal.h"
#include "task_params.cuh"

namespace cqs {

cqs_status make_tmap_bf16(CUtensorMap* m, const void* base, int B, int H, int64_t rows, int D,
                          int64_t sB, int64_t sH, int64_t sN, int box_rows);
void build_task_params_ext(const cqs_plan_t* p, const Task& T, int rows_per_item,
                           const int64_t* src_rows, const int64_t* dst_rows, TaskParams& tp);
cudaError_t launch_attn_bwd_bf16(int D, const CUtensorMap* maps, const TaskParams& tpq,
                                 const TaskParams& tpk, const float* ld, int64_t ld_pitch,
                                 int64_t N, float* dq, float* dk, float* dv, float scale,
                                 cudaStream_t st);
cudaError_t launch_bwd_prep(int D, const void* o, const void* dO, const int64_t* strides,
                            const float* lse, int B, int H, int64_t N, int64_t ld_pitch, float* ld,
                            cudaStream_t st);
cudaError_t launch_merge(int64_t rows, int B, int H, int D, int n_parts, const float* const* po,
                         const float* const* pl, float* acc_o, float* acc_lse, bool acc_write,
                         void* out, cqs_dtype out_dtype, const int64_t* out_strides,
                         int64_t out_row0, int64_t n_total, float* lse_out, cudaStream_t st);

struct BwdLayout {
  int64_t pitch;
  uint64_t ld, dq, dk, dv, total;
};

static BwdLayout bwd_layout(const cqs_plan_desc& d) {
  BwdLayout L;
  const int64_t BH = int64_t(d.B) * d.H;
  L.pitch = (d.N + 3) / 4 * 4;   // 16-byte TMA row pitch
  const uint64_t acc = align256(uint64_t(d.N) * BH * d.D * 4);
  L.ld = 0;
  L.dq = align256(uint64_t(BH) * 2 * L.pitch * 4);
  L.dk = L.dq + acc;
  L.dv = L.dk + acc;
  L.total = L.dv + acc;
  return L;
}

static cqs_status bwd_supported(const cqs_plan_t* p) {
  if (!p) return fail(CQS_E_INVALID, "plan is NULL");
  const cqs_plan_desc& d = p->desc;
  if (d.qkv_loc != CQS_LOC_DEVICE || d.in_dtype != CQS_BF16)
    return fail(CQS_E_UNSUPPORTED, "backward runs resident bf16 plans");
  if (d.D != 64 && d.D != 128) return fail(CQS_E_UNSUPPORTED, "backward head dim must be 64 or 128");
  if (int64_t(d.N) * d.B * d.H >= (int64_t(1) << 31))
    return fail(CQS_E_UNSUPPORTED, "backward: N*B*H must stay below 2^31");
  return CQS_OK;
}

}  // namespace cqs

using namespace cqs;

extern "C" cqs_status cqs_backward_workspace_size(const cqs_plan_t* p, size_t* dev_bytes) {
  if (!dev_bytes) return fail(CQS_E_INVALID, "dev_bytes is NULL");
  cqs_status s = bwd_supported(p);
  if (s != CQS_OK) return s;
  *dev_bytes = size_t(bwd_layout(p->desc).total);
  return CQS_OK;
}

extern "C" cqs_status cqs_backward_partial_view(const cqs_plan_t* p, void* dev_ws, float** dq,
                                                float** dk, float** dv) {
  if (!dev_ws || !dq || !dk || !dv) return fail(CQS_E_INVALID, "NULL argument");
  cqs_status s = bwd_supported(p);
  if (s != CQS_OK) return s;
  const BwdLayout L = bwd_layout(p->desc);
  uint8_t* ws = static_cast<uint8_t*>(dev_ws);
  *dq = reinterpret_cast<float*>(ws + L.dq);
  *dk = reinterpret_cast<float*>(ws + L.dk);
  *dv = reinterpret_cast<float*>(ws + L.dv);
  return CQS_OK;
}

extern "C" cqs_status cqs_attention_backward(const cqs_plan_t* p, const void* q, const void* k,
                                             const void* v, const void* o, const void* dout,
                                             const int64_t qkv_strides[4], const float* lse,
                                             void* dq, void* dk, void* dv,
                                             const int64_t grad_strides[4], float scale,
                                             void* dev_ws, void* stream_, cqs_stats* stats) {
  cqs_status s = bwd_supported(p);
  if (s != CQS_OK) return s;
  const cqs_plan_desc& d = p->desc;
  const bool cast = d.world == 1;   // world > 1: partial accumulators stay in dev_ws
  if (!q || !k || !v || !o || !dout || !lse || !dev_ws || (cast && (!dq || !dk || !dv)))
    return fail(CQS_E_INVALID, "NULL argument");
  if (!qkv_strides || qkv_strides[3] != 1 || (cast && (!grad_strides || grad_strides[3] != 1)))
    return fail(CQS_E_INVALID, "strides: stride(D) must be 1");
  if (reinterpret_cast<uintptr_t>(dev_ws) & 255) return fail(CQS_E_INVALID, "dev_ws must be 256B aligned");
  if ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(dout)) & 15)
    return fail(CQS_E_INVALID, "o/dout must be 16-byte aligned");
  if (scale <= 0.f) scale = 1.f / std::sqrt(float(d.D));
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  const auto t0 = std::chrono::steady_clock::now();
  const BwdLayout L = bwd_layout(d);
  uint8_t* ws = static_cast<uint8_t*>(dev_ws);
  float* ld = reinterpret_cast<float*>(ws + L.ld);
  float* acc_dq = reinterpret_cast<float*>(ws + L.dq);
  float* acc_dk = reinterpret_cast<float*>(ws + L.dk);
  float* acc_dv = reinterpret_cast<float*>(ws + L.dv);

  std::vector<cudaEvent_t> evs;
  auto mark = [&]() {
    if (!stats) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, st);
    evs.push_back(ev);
  };
  int64_t launches = 0, run = 0;
  mark();
  cudaError_t e = launch_bwd_prep(d.D, o, dout, qkv_strides, lse, d.B, d.H, d.N, L.pitch, ld, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(acc_dq, 0, L.total - L.dq, st);
  mark();
  launches += 1;
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("backward prep: ") + cudaGetErrorString(e));

  CUtensorMap maps[4];
  const void* bases[4] = {q, k, v, dout};
  for (int i = 0; i < 4; ++i) {
    s = make_tmap_bf16(&maps[i], bases[i], d.B, d.H, d.N, d.D, qkv_strides[0], qkv_strides[1],
                       qkv_strides[2], 128);
    if (s != CQS_OK) return s;
  }

  TaskParams tpq, tpk;
  for (int64_t ti : p->my_order) {
    const Task& T = p->tasks[size_t(ti)];
    int64_t start[CQS_MAX_SEGS];
    Task Tt = T;   // transposed kept relation: key segment b -> the query segments keeping it
    std::memset(Tt.kept, 0, sizeof(Tt.kept));
    for (int a = 0; a < T.nseg; ++a) {
      start[a] = p->segs[size_t(T.seg_off + a)].start;
      for (int b = 0; b < T.nseg; ++b)
        if (T.kept[a] >> b & 1) Tt.kept[b] |= 1u << a;
    }
    build_task_params_ext(p, T, 128, start, start, tpq);
    build_task_params_ext(p, Tt, 128, start, start, tpk);
    mark();
    e = launch_attn_bwd_bf16(d.D, maps, tpq, tpk, ld, L.pitch, d.N, acc_dq, acc_dk, acc_dv, scale,
                             st);
    mark();
    if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("backward launch: ") + cudaGetErrorString(e));
    launches += 2;
    ++run;
  }
  mark();
  float* accs[3] = {acc_dq, acc_dk, acc_dv};
  void* outs[3] = {dq, dk, dv};
  for (int i = 0; i < 3 && e == cudaSuccess && cast; ++i)
    e = launch_merge(d.N, d.B, d.H, d.D, 0, nullptr, nullptr, accs[i], nullptr, false, outs[i],
                     d.out_dtype, grad_strides, 0, d.N, nullptr, st);
  mark();
  launches += cast ? 3 : 0;
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("backward cast: ") + cudaGetErrorString(e));
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(CQS_E_CUDA, cudaGetErrorString(e));
    stats->ms_total =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (size_t i = 0; i + 1 < evs.size(); i += 2) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, evs[i], evs[i + 1]);
      const bool is_attn = i >= 2 && i < 2 + 2 * size_t(run);
      (is_attn ? stats->ms_attn : stats->ms_merge) += ms;
    }
    for (auto ev : evs) cudaEventDestroy(ev);
    stats->tasks_run = run;
    stats->tasks_skipped = int64_t(p->tasks.size()) - run;
    stats->kernel_launches = launches;
    stats->peak_dev_bytes = L.total;
  }
  return CQS_OK;
}

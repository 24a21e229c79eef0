// Backward executor (Algorithm 2): Delta / lse prep, then for every task of the
// plan the dK/dV and dQ kernels (attn_bwd_sm100.cu) that IndexAdd the task's gradients into fp32
// accumulators, then a cast of the accumulators into the caller's dQ/dK/dV.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
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
                            const float* lse, int64_t lse_pitch, int B, int H, int64_t N,
                            int64_t row0, int64_t ld_pitch, float* ld, cudaStream_t st);
cudaError_t launch_merge(int64_t rows, int B, int H, int D, int n_parts, const float* const* po,
                         const float* const* pl, float* acc_o, float* acc_lse, bool acc_write,
                         void* out, cqs_dtype out_dtype, const int64_t* out_strides,
                         int64_t out_row0, int64_t n_total, float* lse_out, cudaStream_t st);

struct BwdLayout {
  int64_t pitch, F = 0;          // lse/Delta row pitch; streamed: rows per chunk buffer
  int nbuf = 0;                  // streamed: staging buffers
  uint64_t ld, dq, dk, dv, stage = 0, stage_bytes_per_buf = 0, chunk = 0, chunk_bytes = 0,
      chunk_lse = 0, total;
};

// Resident: lse/Delta table [B*H][2][pitch] + three fp32 accumulators [N][B*H][D].
// Streamed (Q/K/V/O/dO/lse and the gradients in pinned host memory): the same table and
// accumulators (the whole N stays on the device: accumulator tier j = 0), plus nbuf staging
// buffers of four tensors [B*H][Lh][D] bf16 (Q, K, V, dO of one task's used segments, Lh = the
// plan's max_staged_rows) and two chunk buffers of F rows that carry O / dO / lse chunks in (prep
// pass) and cast gradient chunks out.
static BwdLayout bwd_layout(const cqs_plan_t* p, int nbuf) {
  const cqs_plan_desc& d = p->desc;
  BwdLayout L;
  const int64_t BH = int64_t(d.B) * d.H, N = d.N, D = d.D;
  L.pitch = (N + 3) / 4 * 4;   // 16-byte rows
  const uint64_t acc = align256(uint64_t(N) * BH * D * 4);
  L.ld = 0;
  L.dq = align256(uint64_t(BH) * 2 * L.pitch * 4);
  L.dk = L.dq + acc;
  L.dv = L.dk + acc;
  L.total = L.dv + acc;
  if (d.qkv_loc == CQS_LOC_PINNED_HOST) {
    L.nbuf = nbuf;
    L.stage = L.total;
    L.stage_bytes_per_buf = 4 * align256(uint64_t(BH) * p->max_staged_rows * D * 2);
    L.chunk = L.stage + uint64_t(nbuf) * L.stage_bytes_per_buf;
    int64_t F = (int64_t(64) << 20) / (BH * D * 4);
    F = std::min<int64_t>(std::max<int64_t>(F, 256), 65536);
    L.F = std::min<int64_t>(F, N);
    L.chunk_lse = align256(uint64_t(L.F) * BH * D * 4);
    L.chunk_bytes = L.chunk_lse + align256(uint64_t(L.F) * BH * 4);
    L.total = L.chunk + 2 * L.chunk_bytes;
  }
  L.total = alloc_bytes(L.total);   // the caller's allocator granularity (R14)
  return L;
}

// Streamed plans: two staging buffers if the budget allows, else one, else infeasible.
static cqs_status bwd_layout_for(const cqs_plan_t* p, BwdLayout* out) {
  if (p->desc.qkv_loc != CQS_LOC_PINNED_HOST) {
    *out = bwd_layout(p, 0);
    return CQS_OK;
  }
  const uint64_t budget = p->desc.budget_bytes;
  for (int nbuf = 2; nbuf >= 1; --nbuf) {
    BwdLayout L = bwd_layout(p, nbuf);
    if (budget == 0 || L.total <= budget) {
      *out = L;
      return CQS_OK;
    }
  }
  return fail(CQS_E_INFEASIBLE,
              "streamed backward: fp32 gradients of all N rows + one staging buffer exceed "
              "budget_bytes at this depth (plan deeper or raise the budget)");
}

static cqs_status bwd_supported(const cqs_plan_t* p) {
  if (!p) return fail(CQS_E_INVALID, "plan is NULL");
  const cqs_plan_desc& d = p->desc;
  if (d.in_dtype != CQS_BF16) return fail(CQS_E_UNSUPPORTED, "backward runs bf16 plans");
  if (d.qkv_loc == CQS_LOC_PINNED_HOST && (d.out_loc != CQS_LOC_PINNED_HOST || d.world != 1))
    return fail(CQS_E_UNSUPPORTED, "streamed backward: single GPU, gradients in pinned host memory");
  if (d.D != 64 && d.D != 128) return fail(CQS_E_UNSUPPORTED, "backward head dim must be 64 or 128");
  if (int64_t(d.N) * d.B * d.H >= (int64_t(1) << 31))
    return fail(CQS_E_UNSUPPORTED, "backward: N*B*H must stay below 2^31");
  return CQS_OK;
}

cqs_status backward_streamed(const cqs_plan_t* p, const BwdLayout& L, const void* q, const void* k,
                             const void* v, const void* o, const void* dout, const float* lse,
                             void* dq, void* dk, void* dv, float scale, uint8_t* ws,
                             cudaStream_t st, cqs_stats* stats);

}  // namespace cqs

using namespace cqs;

extern "C" cqs_status cqs_backward_workspace_size(const cqs_plan_t* p, size_t* dev_bytes) {
  if (!dev_bytes) return fail(CQS_E_INVALID, "dev_bytes is NULL");
  cqs_status s = bwd_supported(p);
  if (s != CQS_OK) return s;
  BwdLayout L;
  if ((s = bwd_layout_for(p, &L)) != CQS_OK) return s;
  *dev_bytes = size_t(L.total);
  return CQS_OK;
}

extern "C" cqs_status cqs_backward_partial_view(const cqs_plan_t* p, void* dev_ws, float** dq,
                                                float** dk, float** dv) {
  if (!dev_ws || !dq || !dk || !dv) return fail(CQS_E_INVALID, "NULL argument");
  cqs_status s = bwd_supported(p);
  if (s != CQS_OK) return s;
  const BwdLayout L = bwd_layout(p, 0);
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
  BwdLayout L;
  if ((s = bwd_layout_for(p, &L)) != CQS_OK) return s;
  if (d.qkv_loc == CQS_LOC_PINNED_HOST) {
    const int64_t c[4] = {int64_t(d.H) * d.N * d.D, int64_t(d.N) * d.D, d.D, 1};
    for (int i = 0; i < 4; ++i)
      if (qkv_strides[i] != c[i] || grad_strides[i] != c[i])
        return fail(CQS_E_INVALID, "streamed backward needs contiguous [B,H,N,D] host tensors");
    return backward_streamed(p, L, q, k, v, o, dout, lse, dq, dk, dv, scale,
                             static_cast<uint8_t*>(dev_ws), st, stats);
  }
  const auto t0 = std::chrono::steady_clock::now();
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
  cudaError_t e = launch_bwd_prep(d.D, o, dout, qkv_strides, lse, d.N, d.B, d.H, d.N, 0, L.pitch,
                                  ld, st);
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
    stats->predicted_peak_bytes = L.total;
  }
  return CQS_OK;
}

// ---------------------------------------------------------------------------------------------
// Streamed backward (Q, K, V, O, dO, lse and the gradients in pinned host memory).  Same
// arithmetic as the resident path; the data path follows the streamed forward (stream.cu):
//   1. prep pass: O / dO / lse rows in chunks of F rows (H2D on a helper stream, double-buffered)
//      -> Delta and -lse*log2e for every row into the device table (global rows);
//   2. per task: the used segments of Q, K, V, dO copied into staging buffer (run mod nbuf) on a
//      copy stream (cudaMemcpy2DAsync, one call per segment per tensor), then the dK/dV and dQ
//      kernels over TMA maps of that buffer, accumulating into the full-N fp32 gradients;
//   3. cast pass: fp32 gradient chunks -> out dtype in a chunk buffer -> D2H on a helper stream.
// ---------------------------------------------------------------------------------------------
namespace cqs {

#define CKB(x)                                                                       \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) return fail(CQS_E_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

cqs_status backward_streamed(const cqs_plan_t* p, const BwdLayout& L, const void* q, const void* k,
                             const void* v, const void* o, const void* dout, const float* lse,
                             void* dq, void* dk, void* dv, float scale, uint8_t* ws,
                             cudaStream_t st, cqs_stats* stats) {
  const cqs_plan_desc& d = p->desc;
  const int64_t N = d.N, D = d.D, BH = int64_t(d.B) * d.H, F = L.F, Lh = p->max_staged_rows;
  const int64_t e_out = d.out_dtype == CQS_BF16 ? 2 : 4;
  const int S = L.nbuf;
  float* ld = reinterpret_cast<float*>(ws + L.ld);
  float* acc[3] = {reinterpret_cast<float*>(ws + L.dq), reinterpret_cast<float*>(ws + L.dk),
                   reinterpret_cast<float*>(ws + L.dv)};
  const uint64_t tens = align256(uint64_t(BH) * Lh * D * 2);
  uint8_t* stage[2][4];
  for (int b = 0; b < S; ++b)
    for (int t = 0; t < 4; ++t) stage[b][t] = ws + L.stage + b * L.stage_bytes_per_buf + t * tens;
  uint8_t* chunk[2] = {ws + L.chunk, ws + L.chunk + L.chunk_bytes};
  const uint8_t* hin[4] = {static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k),
                           static_cast<const uint8_t*>(v), static_cast<const uint8_t*>(dout)};
  const uint8_t* ho = static_cast<const uint8_t*>(o);
  uint8_t* hout[3] = {static_cast<uint8_t*>(dq), static_cast<uint8_t*>(dk),
                      static_cast<uint8_t*>(dv)};

  struct Res {
    cudaStream_t cs = nullptr, fh = nullptr, fd = nullptr;
    std::vector<cudaEvent_t> evs;
    ~Res() {
      for (auto e : evs) cudaEventDestroy(e);
      if (cs) cudaStreamDestroy(cs);
      if (fh) cudaStreamDestroy(fh);
      if (fd) cudaStreamDestroy(fd);
    }
    cudaEvent_t ev() {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      evs.push_back(e);
      return e;
    }
  } R;
  CKB(cudaStreamCreateWithFlags(&R.cs, cudaStreamNonBlocking));   // staging H2D
  CKB(cudaStreamCreateWithFlags(&R.fh, cudaStreamNonBlocking));   // chunk H2D
  CKB(cudaStreamCreateWithFlags(&R.fd, cudaStreamNonBlocking));   // chunk D2H
  cudaEvent_t c_free[2] = {R.ev(), R.ev()}, c_loaded[2] = {R.ev(), R.ev()},
              c_done[2] = {R.ev(), R.ev()};
  cudaEvent_t ev_ready[2] = {R.ev(), R.ev()}, ev_free[2] = {R.ev(), R.ev()};
  bool buf_used[2] = {false, false};
  uint64_t h2d = 0, d2h = 0;
  int64_t launches = 0, run = 0;
  const auto t0 = std::chrono::steady_clock::now();
  // the helper streams start after everything the caller queued on st
  {
    cudaEvent_t start = R.ev();
    CKB(cudaEventRecord(start, st));
    CKB(cudaStreamWaitEvent(R.cs, start, 0));
    CKB(cudaStreamWaitEvent(R.fh, start, 0));
    CKB(cudaStreamWaitEvent(R.fd, start, 0));
  }

  // ---- 1. prep: Delta / -lse*log2e for every row ----
  const int64_t cstr[4] = {int64_t(d.H) * F * D, F * D, D, 1};
  int cb = 0;
  for (int64_t r0 = 0; r0 < N; r0 += F, cb ^= 1) {
    const int64_t n = std::min(F, N - r0);
    uint8_t* co = chunk[cb];
    uint8_t* cdo = chunk[cb] + uint64_t(BH) * F * D * 2;
    float* cl = reinterpret_cast<float*>(chunk[cb] + L.chunk_lse);
    CKB(cudaStreamWaitEvent(R.fh, c_free[cb], 0));
    CKB(cudaMemcpy2DAsync(co, size_t(F * D * 2), ho + r0 * D * 2, size_t(N * D * 2),
                          size_t(n * D * 2), size_t(BH), cudaMemcpyHostToDevice, R.fh));
    CKB(cudaMemcpy2DAsync(cdo, size_t(F * D * 2), hin[3] + r0 * D * 2, size_t(N * D * 2),
                          size_t(n * D * 2), size_t(BH), cudaMemcpyHostToDevice, R.fh));
    CKB(cudaMemcpy2DAsync(cl, size_t(F * 4), lse + r0, size_t(N * 4), size_t(n * 4), size_t(BH),
                          cudaMemcpyHostToDevice, R.fh));
    h2d += uint64_t(BH) * n * (2 * D * 2 + 4);
    CKB(cudaEventRecord(c_loaded[cb], R.fh));
    CKB(cudaStreamWaitEvent(st, c_loaded[cb], 0));
    CKB(launch_bwd_prep(int(D), co, cdo, cstr, cl, F, d.B, d.H, n, r0, L.pitch, ld, st));
    ++launches;
    CKB(cudaEventRecord(c_free[cb], st));
  }
  CKB(cudaMemsetAsync(acc[0], 0, L.stage - L.dq, st));   // the three gradient accumulators
  // staging rows past a task's last used segment feed masked lanes only; keep them finite
  CKB(cudaMemsetAsync(ws + L.stage, 0, size_t(S) * L.stage_bytes_per_buf, st));
  {
    cudaEvent_t zeroed = R.ev();
    CKB(cudaEventRecord(zeroed, st));
    CKB(cudaStreamWaitEvent(R.cs, zeroed, 0));
  }

  // ---- 2. tasks ----
  CUtensorMap maps[2][4];
  for (int b = 0; b < S; ++b)
    for (int t = 0; t < 4; ++t) {
      cqs_status s2 = make_tmap_bf16(&maps[b][t], stage[b][t], d.B, d.H, Lh, d.D,
                                     int64_t(d.H) * Lh * D, Lh * D, D, 128);
      if (s2 != CQS_OK) return s2;
    }
  TaskParams tpq, tpk;
  for (int64_t ti : p->my_order) {
    const Task& T = p->tasks[size_t(ti)];
    const Seg* segs = &p->segs[size_t(T.seg_off)];
    uint32_t used = 0;
    for (int a = 0; a < T.nseg; ++a)
      if (T.kept[a]) used |= (1u << a) | T.kept[a];
    int64_t src[CQS_MAX_SEGS], dst[CQS_MAX_SEGS], off = 0;
    for (int a = 0; a < T.nseg; ++a) {
      src[a] = off;
      dst[a] = segs[a].start;
      if (used >> a & 1) off += segs[a].len;
    }
    const int b = int(run % S);
    if (buf_used[b]) CKB(cudaStreamWaitEvent(R.cs, ev_free[b], 0));
    for (int a = 0; a < T.nseg; ++a) {
      if (!(used >> a & 1)) continue;
      for (int t = 0; t < 4; ++t)
        CKB(cudaMemcpy2DAsync(stage[b][t] + src[a] * D * 2, size_t(Lh * D * 2),
                              hin[t] + segs[a].start * D * 2, size_t(N * D * 2),
                              size_t(segs[a].len * D * 2), size_t(BH), cudaMemcpyHostToDevice,
                              R.cs));
      h2d += uint64_t(4 * segs[a].len * D * 2 * BH);
    }
    CKB(cudaEventRecord(ev_ready[b], R.cs));
    CKB(cudaStreamWaitEvent(st, ev_ready[b], 0));
    Task Tt = T;
    std::memset(Tt.kept, 0, sizeof(Tt.kept));
    for (int a = 0; a < T.nseg; ++a)
      for (int c = 0; c < T.nseg; ++c)
        if (T.kept[a] >> c & 1) Tt.kept[c] |= 1u << a;
    build_task_params_ext(p, T, 128, src, dst, tpq);
    build_task_params_ext(p, Tt, 128, src, dst, tpk);
    CKB(launch_attn_bwd_bf16(int(D), maps[b], tpq, tpk, ld, L.pitch, N, acc[0], acc[1], acc[2],
                             scale, st));
    launches += 2;
    CKB(cudaEventRecord(ev_free[b], st));
    buf_used[b] = true;
    ++run;
  }

  // ---- 3. cast + D2H ----
  const int64_t ostr[4] = {int64_t(d.H) * F * D, F * D, D, 1};
  for (int g = 0; g < 3; ++g)
    for (int64_t r0 = 0; r0 < N; r0 += F, cb ^= 1) {
      const int64_t n = std::min(F, N - r0);
      CKB(cudaStreamWaitEvent(st, c_free[cb], 0));
      CKB(launch_merge(n, d.B, d.H, d.D, 0, nullptr, nullptr, acc[g] + r0 * BH * D, nullptr, false,
                       chunk[cb], d.out_dtype, ostr, 0, F, nullptr, st));
      ++launches;
      CKB(cudaEventRecord(c_done[cb], st));
      CKB(cudaStreamWaitEvent(R.fd, c_done[cb], 0));
      CKB(cudaMemcpy2DAsync(hout[g] + r0 * D * e_out, size_t(N * D * e_out), chunk[cb],
                            size_t(F * D * e_out), size_t(n * D * e_out), size_t(BH),
                            cudaMemcpyDeviceToHost, R.fd));
      d2h += uint64_t(BH) * n * D * e_out;
      CKB(cudaEventRecord(c_free[cb], R.fd));
    }
  {   // the caller's stream covers every copy issued on the helper streams
    cudaEvent_t e1 = R.ev(), e2 = R.ev(), e3 = R.ev();
    CKB(cudaEventRecord(e1, R.fd));
    CKB(cudaEventRecord(e2, R.fh));
    CKB(cudaEventRecord(e3, R.cs));
    CKB(cudaStreamWaitEvent(st, e1, 0));
    CKB(cudaStreamWaitEvent(st, e2, 0));
    CKB(cudaStreamWaitEvent(st, e3, 0));
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    CKB(cudaStreamSynchronize(st));
    stats->ms_total =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    stats->bytes_h2d = h2d;
    stats->bytes_d2h = d2h;
    stats->tasks_run = run;
    stats->tasks_skipped = int64_t(p->tasks.size()) - run;
    stats->kernel_launches = launches;
    stats->predicted_peak_bytes = L.total;
  }
  return CQS_OK;
}

}  // namespace cqs

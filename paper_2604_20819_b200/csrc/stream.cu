// Streamed forward: Q/K/V (and O, lse) in pinned host memory, QKV larger than the device budget
// (Sec. 2.4-2.5 P:145-162 "scale beyond the memory limits of a single device", Sec. 4
// P:244 "continuously pipelined between host and device").
//
// Per task (leaf) the segments that carry kept work are copied H2D (cudaMemcpy2DAsync: rows = the
// B*H planes, pitch N*D) into staging buffer t mod S on a copy stream while task t-1 computes
// (S = 2: double buffering).  The attention kernel addresses the staged segments through TMA maps
// over the staging buffer.  Partials are LSE-merged into a device accumulator that covers one
// depth-j subtree (all rows of one depth-j intermediate subsequence; j = plan acc_depth).  When a
// subtree is done its accumulator is merged into the pinned-host fp32 accumulator (H2D chunk ->
// cqs_merge kernel -> D2H), and a final pass converts the host accumulator to O / lse.  With j = 0
// the device accumulator covers all N rows and is finalized directly.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
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
cudaError_t launch_merge(int64_t rows, int B, int H, int D, int n_parts, const float* const* po,
                         const float* const* pl, float* acc_o, float* acc_lse, bool acc_write,
                         void* out, cqs_dtype out_dtype, const int64_t* out_strides,
                         int64_t out_row0, int64_t n_total, float* lse_out, cudaStream_t st);
cqs_status make_tmap_bf16(CUtensorMap* m, const void* base, int B, int H, int64_t rows, int D,
                          int64_t sB, int64_t sH, int64_t sN, int box_rows);
int attn_rows_per_item(int D);
int attn_box_rows(int D, int which);
void build_task_params_ext(const cqs_plan_t* p, const Task& T, int rows_per_item,
                           const int64_t* src_rows, const int64_t* dst_rows, TaskParams& tp);
void build_task_params_raw(int BH, int H, int nseg, const int64_t* len, const uint32_t* kept,
                           int rows_per_item, const int64_t* src_rows, const int64_t* dst_rows,
                           TaskParams& tp);

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) return fail(CQS_E_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

// Pieces per segment of the first task (staged and launched as they land) and per active query
// segment of the last task (downloaded while the next piece computes).  Measured on C2 e2e: one
// piece per segment 263 ms / step, four pieces 275 ms (each extra launch of a partial block adds a
// wave-quantisation tail that costs more than the shorter fill / drain saves).
constexpr int kFirstPieces = 1;
constexpr int kLastPieces = 1;

namespace {
struct Scoped {
  cudaStream_t cs = nullptr, fh = nullptr, fd = nullptr;
  std::vector<cudaEvent_t> evs;
  ~Scoped() {
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
};
}  // namespace

cqs_status forward_streamed(const cqs_plan_t* p, const void* q, const void* k, const void* v,
                            void* out, const int64_t* out_strides, float* lse, float scale,
                            uint8_t* ws, uint8_t* host_ws, cudaStream_t st, cqs_stats* stats) {
  const cqs_plan_desc& d = p->desc;
  if (d.out_loc != CQS_LOC_PINNED_HOST)
    return fail(CQS_E_UNSUPPORTED, "streamed Q/K/V require a pinned-host output");
  // world > 1: this rank stages only its tasks' segments and keeps its partials in the rank-local
  // device accumulator (held blocks, acc_depth 0); the exchange (cqs_exchange_merge) finalizes
  const bool sharded = d.world > 1;
  const int64_t N = d.N, D = d.D, BH = int64_t(d.B) * d.H;
  if (!sharded && (out_strides[0] != int64_t(d.H) * N * D || out_strides[1] != N * D ||
                   out_strides[2] != D))
    return fail(CQS_E_INVALID, "streamed mode needs a contiguous [B,H,N,D] output");
  const int64_t e_in = d.in_dtype == CQS_BF16 ? 2 : 4, e_out = d.out_dtype == CQS_BF16 ? 2 : 4;
  const int S = p->n_stage_buffers, j = p->acc_depth;
  const int64_t Lh = p->max_staged_rows, Lacc = p->max_acc_rows;
  const WsLayout L = ws_layout(d, Lh, Lacc, S);
  float* acc_o = reinterpret_cast<float*>(ws + L.acc_o);
  float* acc_l = reinterpret_cast<float*>(ws + L.acc_lse);
  const uint64_t tens_bytes = align256(uint64_t(BH * Lh * D * e_in));
  uint8_t* stage[2][3];
  for (int b = 0; b < S; ++b)
    for (int t = 0; t < 3; ++t) stage[b][t] = ws + L.stage + b * L.stage_bytes_per_buf + t * tens_bytes;
  const int64_t F = flush_rows(Lacc, BH, D);
  const uint64_t fbo = align256(uint64_t(F * BH * D * 4)), fbl = align256(uint64_t(F * BH * 4));
  float* fb_o[2];
  float* fb_l[2];
  for (int i = 0; i < 2; ++i) {
    fb_o[i] = reinterpret_cast<float*>(ws + L.flush + i * (fbo + fbl));
    fb_l[i] = reinterpret_cast<float*>(ws + L.flush + i * (fbo + fbl) + fbo);
  }
  float* hacc_o = reinterpret_cast<float*>(host_ws);
  float* hacc_l = host_ws ? reinterpret_cast<float*>(host_ws + align256(uint64_t(N * BH * D * 4)))
                          : nullptr;
  const uint8_t* hq[3] = {static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k),
                          static_cast<const uint8_t*>(v)};

  Scoped sc;
  CK(cudaStreamCreateWithFlags(&sc.cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sc.fh, cudaStreamNonBlocking));   // flush H2D
  CK(cudaStreamCreateWithFlags(&sc.fd, cudaStreamNonBlocking));   // flush / output D2H
  // flush buffer b: loaded (H2D done) -> merged (kernel done) -> free (D2H done)
  cudaEvent_t fb_loaded[2] = {sc.ev(), sc.ev()}, fb_merged[2] = {sc.ev(), sc.ev()},
              fb_free[2] = {sc.ev(), sc.ev()};
  int fb_next = 0;
  cudaEvent_t flush_done = sc.ev();
  bool flushed_once = false;
  cudaEvent_t ev_ready[2] = {sc.ev(), sc.ev()}, ev_free[2] = {sc.ev(), sc.ev()};
  bool buf_used[2] = {false, false};
  uint64_t h2d = 0, d2h = 0;
  int64_t launches = 0, run = 0;
  const auto t0 = std::chrono::steady_clock::now();

  CUtensorMap maps[2][3];
  if (d.in_dtype == CQS_BF16)
    for (int b = 0; b < S; ++b)
      for (int t = 0; t < 3; ++t) {
        cqs_status s2 = make_tmap_bf16(&maps[b][t], stage[b][t], d.B, d.H, Lh, d.D,
                                       int64_t(d.H) * Lh * D, Lh * D, D,
                                       attn_box_rows(d.D, t));
        if (s2 != CQS_OK) return s2;
      }
  const int64_t sstr[4] = {int64_t(d.H) * Lh * D, Lh * D, D, 1};

  // Flush-buffer pipeline (two buffers alternate): H2D on sc.fh, kernel on st, D2H on sc.fd, so
  // chunk i+1's upload, chunk i's merge and chunk i-1's download overlap.
  auto fb_acquire = [&]() -> int {
    const int b = fb_next;
    fb_next ^= 1;
    cudaStreamWaitEvent(sc.fh, fb_free[b], 0);   // never-recorded events are no-ops
    cudaStreamWaitEvent(st, fb_free[b], 0);
    return b;
  };
  // final O/lse for rows [r0, r0+n) from an fp32 [n][BH][D] + [n][BH] source on the device,
  // staged as [BH][F][D] out + [BH][F] lse in flush buffer `b` and downloaded on sc.fd
  // (with part_o / part_l: the final rows are the LSE merge of that partial and src)
  auto emit_final = [&](int b, const float* src_o, const float* src_l, int64_t r0, int64_t n,
                        const float* part_o = nullptr, const float* part_l = nullptr) -> cqs_status {
    const int64_t ostr[4] = {int64_t(d.H) * F * D, F * D, D, 1};
    void* ob = fb_o[b];
    float* lb = fb_l[b];
    CK(launch_merge(n, d.B, d.H, d.D, part_o ? 1 : 0, part_o ? &part_o : nullptr,
                    part_l ? &part_l : nullptr, const_cast<float*>(src_o),
                    const_cast<float*>(src_l), false, ob, d.out_dtype, ostr, 0, F, lb, st));
    ++launches;
    CK(cudaEventRecord(fb_merged[b], st));
    CK(cudaStreamWaitEvent(sc.fd, fb_merged[b], 0));
    CK(cudaMemcpy2DAsync(static_cast<uint8_t*>(out) + r0 * D * e_out, size_t(N * D * e_out), ob,
                         size_t(F * D * e_out), size_t(n * D * e_out), size_t(BH),
                         cudaMemcpyDeviceToHost, sc.fd));
    d2h += uint64_t(n * D * e_out * BH);
    if (lse) {
      CK(cudaMemcpy2DAsync(lse + r0, size_t(N * 4), lb, size_t(F * 4), size_t(n * 4), size_t(BH),
                           cudaMemcpyDeviceToHost, sc.fd));
      d2h += uint64_t(n * 4 * BH);
    }
    CK(cudaEventRecord(fb_free[b], sc.fd));
    return CQS_OK;
  };

  // Staging rows past a task's last staged segment are read by the last key tile of a segment
  // (masked to P = 0) — they must be finite, since 0 * NaN = NaN in the P.V MMA.  Zero once.
  CK(cudaMemsetAsync(ws + L.stage, 0, size_t(S) * L.stage_bytes_per_buf, st));
  {
    cudaEvent_t zeroed = sc.ev();   // the copy stream must not stage before the zeroing
    CK(cudaEventRecord(zeroed, st));
    CK(cudaStreamWaitEvent(sc.cs, zeroed, 0));
  }

  if (j > 0) {  // host accumulator starts empty: lse = -inf
    CK(launch_fill(fb_l[0], F * BH, -INFINITY, st));
    ++launches;
    for (int64_t r = 0; r < N; r += F) {
      const int64_t n = std::min(F, N - r);
      CK(cudaMemcpyAsync(hacc_l + r * BH, fb_l[0], size_t(n * BH * 4), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaEventRecord(fb_free[0], st));     // flush buffer 0 and the host rows are settled
    CK(cudaStreamWaitEvent(sc.fh, fb_free[0], 0));
  }

  std::vector<Seg> node;
  int64_t gi = 0;
  const int64_t nmy = int64_t(p->my_order.size());

  // Device-tier accumulator (j = 0): a row is final after the last task that merges into it (its
  // segment is an active query segment of that task), so its O / lse are converted and downloaded
  // right after that task instead of after the whole tree — the output D2H overlaps the remaining
  // tasks (at depth 1, 4 of the 7 chunks are final before the last task).  fin[ti] = the row
  // ranges whose last task is ti, from a sweep over the active query segments of every task.
  std::vector<std::vector<std::pair<int64_t, int64_t>>> fin;
  if (j == 0 && nmy > 0 && !sharded) {
    std::vector<std::pair<int64_t, int64_t>> ev;   // (row, +(ti+1) at start / -(ti+1) at end)
    for (int64_t ti = 0; ti < nmy; ++ti) {
      const Task& T = p->tasks[size_t(p->my_order[size_t(ti)])];
      const Seg* sg = &p->segs[size_t(T.seg_off)];
      for (int a = 0; a < T.nseg; ++a)
        if (T.kept[a] && sg[a].len > 0) {
          ev.push_back({sg[a].start, ti + 1});
          ev.push_back({sg[a].start + sg[a].len, -(ti + 1)});
        }
    }
    std::sort(ev.begin(), ev.end());
    std::vector<int64_t> open_cnt(size_t(nmy) + 1, 0);   // covering tasks, by index
    std::vector<int64_t> heap;                            // max-heap of open task indices
    fin.assign(size_t(nmy), {});
    int64_t row = 0;
    size_t e = 0;
    while (row < N) {
      while (e < ev.size() && ev[e].first <= row) {       // apply every event at `row`
        const int64_t t = ev[e].second;
        if (t > 0) {
          if (open_cnt[size_t(t)]++ == 0) {
            heap.push_back(t);
            std::push_heap(heap.begin(), heap.end());
          }
        } else {
          --open_cnt[size_t(-t)];
        }
        ++e;
      }
      while (!heap.empty() && open_cnt[size_t(heap.front())] == 0) {
        std::pop_heap(heap.begin(), heap.end());
        heap.pop_back();
      }
      const int64_t next = e < ev.size() ? std::min<int64_t>(ev[e].first, N) : N;
      // rows no task of this rank touches (none at world 1) are emitted after the last task
      const int64_t last = heap.empty() ? nmy : heap.front();
      auto& v = fin[size_t(last - 1)];
      if (!v.empty() && v.back().first + v.back().second == row)
        v.back().second += next - row;
      else
        v.push_back({row, next - row});
      row = next;
    }
  }
  // Host-tier accumulators (j > 0): a row is final after the flush of the last depth-j subtree
  // that contains it; at that flush its merged value is converted and downloaded straight from the
  // flush buffers instead of being written back to the host accumulator and re-read by a final
  // pass.  fin_g[g] = the row ranges whose last subtree is g (same sweep as fin, over the nodes).
  std::vector<std::vector<std::pair<int64_t, int64_t>>> fin_g;
  // first_g[g] = the row ranges whose FIRST subtree is g: the host accumulator holds nothing for
  // them yet, so their flush is a plain copy of the device rows (no host upload, no merge)
  std::vector<std::vector<std::pair<int64_t, int64_t>>> first_g;
  bool direct_final = false;
  if (j > 0 && nmy > 0) {
    std::vector<std::pair<int64_t, int64_t>> ev;
    int64_t ng = 0;
    std::vector<Seg> nd;
    for (int64_t g0 = 0; g0 < nmy; ++ng) {
      const Task& A = p->tasks[size_t(p->my_order[size_t(g0)])];
      int64_t g1 = g0 + 1;
      while (g1 < nmy &&
             std::equal(A.quorum, A.quorum + j, p->tasks[size_t(p->my_order[size_t(g1)])].quorum))
        ++g1;
      build_segments(N, p->lv, A.quorum, j, nd);
      for (const Seg& sg : nd)
        if (sg.len > 0) {
          ev.push_back({sg.start, ng + 1});
          ev.push_back({sg.start + sg.len, -(ng + 1)});
        }
      g0 = g1;
    }
    std::sort(ev.begin(), ev.end());
    std::vector<int64_t> open_cnt(size_t(ng) + 1, 0), heap, heap_min;
    fin_g.assign(size_t(ng), {});
    first_g.assign(size_t(ng), {});
    direct_final = true;
    int64_t row = 0;
    size_t e = 0;
    while (row < N) {
      while (e < ev.size() && ev[e].first <= row) {
        const int64_t t = ev[e].second;
        if (t > 0) {
          if (open_cnt[size_t(t)]++ == 0) {
            heap.push_back(t);
            std::push_heap(heap.begin(), heap.end());
            heap_min.push_back(t);
            std::push_heap(heap_min.begin(), heap_min.end(), std::greater<int64_t>());
          }
        } else {
          --open_cnt[size_t(-t)];
        }
        ++e;
      }
      while (!heap.empty() && open_cnt[size_t(heap.front())] == 0) {
        std::pop_heap(heap.begin(), heap.end());
        heap.pop_back();
      }
      while (!heap_min.empty() && open_cnt[size_t(heap_min.front())] == 0) {
        std::pop_heap(heap_min.begin(), heap_min.end(), std::greater<int64_t>());
        heap_min.pop_back();
      }
      const int64_t next = e < ev.size() ? std::min<int64_t>(ev[e].first, N) : N;
      if (heap.empty()) {
        // a row in no subtree: only with CQS_PLAN_SUBSET (a full tree at world 1 covers every
        // row); such rows are left unwritten — reading the host accumulator for them would touch
        // all of it
      } else {
        auto& v = fin_g[size_t(heap.front() - 1)];
        if (!v.empty() && v.back().first + v.back().second == row)
          v.back().second += next - row;
        else
          v.push_back({row, next - row});
        auto& w = first_g[size_t(heap_min.front() - 1)];
        if (!w.empty() && w.back().first + w.back().second == row)
          w.back().second += next - row;
        else
          w.push_back({row, next - row});
      }
      row = next;
    }
  }
  int64_t gidx = 0;   // subtree counter of the main loop (j > 0)
  auto emit_rows = [&](int64_t r0, int64_t len) -> cqs_status {   // j = 0: acc row = global row
    for (int64_t c0 = 0; c0 < len; c0 += F) {
      const int64_t n = std::min(F, len - c0);
      cqs_status s2 = emit_final(fb_acquire(), acc_o + (r0 + c0) * BH * D,
                                 acc_l + (r0 + c0) * BH, r0 + c0, n);
      if (s2 != CQS_OK) return s2;
    }
    return CQS_OK;
  };
  while (gi < nmy) {
    // ---- one depth-j subtree: tasks sharing quorum prefix (q_1..q_j) ----
    const Task& T0 = p->tasks[size_t(p->my_order[size_t(gi)])];
    int64_t ge = gi + 1;
    while (ge < nmy &&
           std::equal(T0.quorum, T0.quorum + j, p->tasks[size_t(p->my_order[size_t(ge)])].quorum))
      ++ge;
    build_segments(N, p->lv, T0.quorum, j, node);
    std::vector<int64_t> node_off(node.size());
    int64_t node_rows = 0;
    for (size_t i = 0; i < node.size(); ++i) node_off[i] = node_rows, node_rows += node[i].len;
    CK(launch_fill(acc_l, (sharded ? Lacc : node_rows) * BH, -INFINITY, st));
    ++launches;

    for (int64_t ti = gi; ti < ge; ++ti) {
      const Task& T = p->tasks[size_t(p->my_order[size_t(ti)])];
      const Seg* segs = &p->segs[size_t(T.seg_off)];
      uint32_t used = 0;
      for (int a = 0; a < T.nseg; ++a)
        if (T.kept[a]) used |= (1u << a) | T.kept[a];
      int64_t src[CQS_MAX_SEGS], dst[CQS_MAX_SEGS], off = 0;
      for (int a = 0; a < T.nseg; ++a) {
        src[a] = off;
        if (used >> a & 1) off += segs[a].len;
        size_t s = 0;
        while (s + 1 < node.size() &&
               !(segs[a].start >= node[s].start && segs[a].start < node[s].start + node[s].len))
          ++s;
        dst[a] = sharded ? p->acc_row(segs[a].start) : node_off[s] + (segs[a].start - node[s].start);
      }
      const int b = int(run % S);
      if (buf_used[b]) CK(cudaStreamWaitEvent(sc.cs, ev_free[b], 0));
      auto launch = [&](const Task& Tl) -> cqs_status {
        TaskParams tp;
        build_task_params_ext(p, Tl, d.in_dtype == CQS_BF16 ? attn_rows_per_item(d.D) : 32, src,
                              dst, tp);
        if (d.in_dtype == CQS_BF16)
          CK(launch_attn_bf16(d.D, maps[b], tp, acc_o, acc_l, scale, st));
        else
          CK(launch_attn_f32(d.D, tp, reinterpret_cast<const float*>(stage[b][0]),
                             reinterpret_cast<const float*>(stage[b][1]),
                             reinterpret_cast<const float*>(stage[b][2]), sstr, acc_o, acc_l,
                             scale, st));
        ++launches;
        return CQS_OK;
      };
      // The first task has nothing to overlap its staging with, so it runs piece by piece as its
      // data lands: after piece x arrives, one launch covers the kept (query, key) piece pairs
      // whose later piece is x.  Splitting a task's key set over launches is exact: each launch
      // LSE-merges its partial into the accumulator like a task (Eq. 3).
      const bool split_first = run == 0;
      if (split_first) {
        // pieces: every used segment cut into up to 4 consecutive row ranges (multiples of the
        // 128-row tile, >= 2048 rows each) so the first launch waits for a quarter of a segment;
        // a piece pair is kept iff its parent segments' pair is (pieces of one segment share its
        // per-level codes, so the CQS mask is unchanged)
        const int rpi = d.in_dtype == CQS_BF16 ? attn_rows_per_item(d.D) : 32;
        const int nused = __builtin_popcount(used);
        const int pmax = std::max(1, std::min(kFirstPieces, CQS_MAX_SEGS / nused));
        int64_t pl[CQS_MAX_SEGS], ps[CQS_MAX_SEGS], psrc[CQS_MAX_SEGS], pdst[CQS_MAX_SEGS];
        int par[CQS_MAX_SEGS], np = 0;
        for (int a = 0; a < T.nseg; ++a) {
          if (!(used >> a & 1)) continue;
          const int64_t L = segs[a].len;
          int k = int(std::min<int64_t>(pmax, std::max<int64_t>(1, L / 2048)));
          const int64_t step = (L / k + 127) / 128 * 128;
          for (int64_t o = 0; o < L; o += step) {
            pl[np] = std::min(step, L - o);
            ps[np] = segs[a].start + o;
            psrc[np] = src[a] + o;
            pdst[np] = dst[a] + o;
            par[np] = a;
            ++np;
          }
        }
        uint32_t pk[CQS_MAX_SEGS] = {};
        for (int x = 0; x < np; ++x)
          for (int y = 0; y < np; ++y)
            if (T.kept[par[x]] >> par[y] & 1) pk[x] |= 1u << y;
        uint32_t arrived = 0;
        for (int x = 0; x < np; ++x) {
          for (int t = 0; t < 3; ++t)
            CK(cudaMemcpy2DAsync(stage[b][t] + psrc[x] * D * e_in, size_t(Lh * D * e_in),
                                 hq[t] + ps[x] * D * e_in, size_t(N * D * e_in),
                                 size_t(pl[x] * D * e_in), size_t(BH), cudaMemcpyHostToDevice,
                                 sc.cs));
          h2d += uint64_t(3 * pl[x] * D * e_in * BH);
          arrived |= 1u << x;
          uint32_t kx[CQS_MAX_SEGS];
          bool any = false;
          for (int y = 0; y < np; ++y) {
            kx[y] = y == x ? pk[y] & arrived : ((arrived >> y & 1) ? pk[y] & (1u << x) : 0u);
            any |= kx[y] != 0;
          }
          if (!any) continue;
          cudaEvent_t piece_ready = sc.ev();
          CK(cudaEventRecord(piece_ready, sc.cs));
          CK(cudaStreamWaitEvent(st, piece_ready, 0));
          TaskParams tp;
          build_task_params_raw(d.B * d.H, d.H, np, pl, kx, rpi, psrc, pdst, tp);
          if (d.in_dtype == CQS_BF16)
            CK(launch_attn_bf16(d.D, maps[b], tp, acc_o, acc_l, scale, st));
          else
            CK(launch_attn_f32(d.D, tp, reinterpret_cast<const float*>(stage[b][0]),
                               reinterpret_cast<const float*>(stage[b][1]),
                               reinterpret_cast<const float*>(stage[b][2]), sstr, acc_o, acc_l,
                               scale, st));
          ++launches;
        }
      }
      for (int a = 0; a < T.nseg && !split_first; ++a) {
        if (!(used >> a & 1)) continue;
        for (int t = 0; t < 3; ++t)
          CK(cudaMemcpy2DAsync(stage[b][t] + src[a] * D * e_in, size_t(Lh * D * e_in),
                               hq[t] + segs[a].start * D * e_in, size_t(N * D * e_in),
                               size_t(segs[a].len * D * e_in), size_t(BH),
                               cudaMemcpyHostToDevice, sc.cs));
        h2d += uint64_t(3 * segs[a].len * D * e_in * BH);
      }
      // The last task has nothing after it to overlap the output download with, so it runs query
      // piece by query piece (up to 4 per active query segment) and each piece's final rows are
      // downloaded while the next piece computes (device-tier accumulator only).
      const bool split_last = j == 0 && !sharded && !split_first && ti == nmy - 1;
      if (!split_first) {
        CK(cudaEventRecord(ev_ready[b], sc.cs));
        CK(cudaStreamWaitEvent(st, ev_ready[b], 0));
        if (!split_last) {
          cqs_status s2 = launch(T);
          if (s2 != CQS_OK) return s2;
        }
      }
      std::vector<std::pair<int64_t, int64_t>> rest;   // final rows of this task still to emit
      if (j == 0 && !sharded) rest = fin[size_t(ti)];
      // query pieces of the last task (up to 4 per active query segment, multiples of the
      // work-item rows): a piece's rows are downloaded while the next piece computes
      const int rpi_l = d.in_dtype == CQS_BF16 ? attn_rows_per_item(d.D) : 32;
      int64_t lq_len[CQS_MAX_SEGS], lq_src[CQS_MAX_SEGS], lq_dst[CQS_MAX_SEGS];
      for (int x = 0; x < T.nseg; ++x)
        lq_len[x] = segs[x].len, lq_src[x] = src[x], lq_dst[x] = dst[x];
      if (split_last)
        for (int a = 0; a < T.nseg; ++a) {
          if (!T.kept[a]) continue;
          const int npc = std::max(1, std::min<int>(kLastPieces, CQS_MAX_SEGS - T.nseg));
          const int64_t L = segs[a].len;
          const int k = int(std::min<int64_t>(npc, std::max<int64_t>(1, L / 4096)));
          const int64_t step = (L / k + rpi_l - 1) / rpi_l * rpi_l;
          for (int64_t o = 0; o < L; o += step) {
            // the piece is segment T.nseg (appended): query rows [o, o + len) of segment a
            const int nq = T.nseg;
            lq_len[nq] = std::min(step, L - o);
            lq_src[nq] = src[a] + o;
            lq_dst[nq] = dst[a] + o;
            uint32_t kx[CQS_MAX_SEGS] = {};
            kx[nq] = T.kept[a];
            TaskParams tp;
            build_task_params_raw(d.B * d.H, d.H, nq + 1, lq_len, kx, rpi_l, lq_src, lq_dst, tp);
            if (d.in_dtype == CQS_BF16)
              CK(launch_attn_bf16(d.D, maps[b], tp, acc_o, acc_l, scale, st));
            else
              CK(launch_attn_f32(d.D, tp, reinterpret_cast<const float*>(stage[b][0]),
                                 reinterpret_cast<const float*>(stage[b][1]),
                                 reinterpret_cast<const float*>(stage[b][2]), sstr, acc_o, acc_l,
                                 scale, st));
            ++launches;
            // rows of this piece whose last task is this one: emit them now, keep the remainder
            const int64_t lo = segs[a].start + o, hi = lo + lq_len[nq];
            std::vector<std::pair<int64_t, int64_t>> keep;
            for (const auto& iv : rest) {
              const int64_t s0 = std::max(iv.first, lo), s1 = std::min(iv.first + iv.second, hi);
              if (s0 >= s1) {
                keep.push_back(iv);
                continue;
              }
              cqs_status s2 = emit_rows(s0, s1 - s0);
              if (s2 != CQS_OK) return s2;
              if (iv.first < s0) keep.push_back({iv.first, s0 - iv.first});
              if (s1 < iv.first + iv.second) keep.push_back({s1, iv.first + iv.second - s1});
            }
            rest.swap(keep);
          }
        }
      CK(cudaEventRecord(ev_free[b], st));
      buf_used[b] = true;
      ++run;
      for (const auto& iv : rest) {
        cqs_status s2 = emit_rows(iv.first, iv.second);
        if (s2 != CQS_OK) return s2;
      }
    }

    // ---- flush the subtree accumulator (pipelined over the two flush buffers) ----
    if (j > 0 && flushed_once) CK(cudaStreamWaitEvent(sc.fh, flush_done, 0));  // host rows settled
    const std::vector<std::pair<int64_t, int64_t>>* fg =
        direct_final ? &fin_g[size_t(gidx)] : nullptr;
    const std::vector<std::pair<int64_t, int64_t>>* ff =
        direct_final ? &first_g[size_t(gidx)] : nullptr;
    // is `grow` inside one of the sorted disjoint intervals iv? cuts n at the next boundary
    auto in_ranges = [](const std::vector<std::pair<int64_t, int64_t>>* iv, int64_t grow,
                        int64_t& n) {
      // node segments come in the node's chunk order (I order), not in row order: look up the
      // first interval that ends after `grow`
      size_t k = size_t(std::upper_bound(iv->begin(), iv->end(), grow,
                                         [](int64_t r, const std::pair<int64_t, int64_t>& x) {
                                           return r < x.first + x.second;
                                         }) - iv->begin());
      if (k < iv->size() && (*iv)[k].first <= grow) {
        n = std::min(n, (*iv)[k].first + (*iv)[k].second - grow);
        return true;
      }
      if (k < iv->size()) n = std::min(n, (*iv)[k].first - grow);
      return false;
    };
    for (size_t s = 0; s < node.size() && j > 0; ++s) {   // (j = 0: emitted task by task above)
      for (int64_t c0 = 0; c0 < node[s].len;) {
        const int64_t grow = node[s].start + c0, lrow = node_off[s] + c0;
        int64_t n = std::min(F, node[s].len - c0);
        const bool final_rows = fg && in_ranges(fg, grow, n);   // last subtree of these rows
        const bool first_rows = ff && in_ranges(ff, grow, n);   // first subtree of these rows
        c0 += n;
        const float* po = acc_o + lrow * BH * D;
        const float* pl = acc_l + lrow * BH;
        if (first_rows && final_rows) {   // only subtree of these rows: final straight from acc
          cqs_status s2 = emit_final(fb_acquire(), po, pl, grow, n);
          if (s2 != CQS_OK) return s2;
          continue;
        }
        if (first_rows) {   // nothing in the host rows yet: copy the device rows out
          const int b = fb_acquire();
          CK(cudaMemcpyAsync(fb_o[b], po, size_t(n * BH * D * 4), cudaMemcpyDeviceToDevice, st));
          CK(cudaMemcpyAsync(fb_l[b], pl, size_t(n * BH * 4), cudaMemcpyDeviceToDevice, st));
          CK(cudaEventRecord(fb_merged[b], st));
          CK(cudaStreamWaitEvent(sc.fd, fb_merged[b], 0));
          CK(cudaMemcpyAsync(hacc_o + grow * BH * D, fb_o[b], size_t(n * BH * D * 4),
                             cudaMemcpyDeviceToHost, sc.fd));
          CK(cudaMemcpyAsync(hacc_l + grow * BH, fb_l[b], size_t(n * BH * 4),
                             cudaMemcpyDeviceToHost, sc.fd));
          CK(cudaEventRecord(fb_free[b], sc.fd));
          d2h += uint64_t(n * BH * (D + 1) * 4);
          continue;
        }
        const int b = fb_acquire();
        CK(cudaMemcpyAsync(fb_o[b], hacc_o + grow * BH * D, size_t(n * BH * D * 4),
                           cudaMemcpyHostToDevice, sc.fh));
        CK(cudaMemcpyAsync(fb_l[b], hacc_l + grow * BH, size_t(n * BH * 4),
                           cudaMemcpyHostToDevice, sc.fh));
        CK(cudaEventRecord(fb_loaded[b], sc.fh));
        CK(cudaStreamWaitEvent(st, fb_loaded[b], 0));
        h2d += uint64_t(n * BH * (D + 1) * 4);
        if (final_rows) {   // merge + convert into the other flush buffer, download O / lse
          cqs_status s2 = emit_final(fb_acquire(), fb_o[b], fb_l[b], grow, n, po, pl);
          if (s2 != CQS_OK) return s2;
          CK(cudaEventRecord(fb_free[b], st));   // input consumed by the merge kernel
          continue;
        }
        CK(launch_merge(n, d.B, d.H, d.D, 1, &po, &pl, fb_o[b], fb_l[b], true, nullptr,
                        d.out_dtype, nullptr, 0, n, nullptr, st));
        ++launches;
        CK(cudaEventRecord(fb_merged[b], st));
        CK(cudaStreamWaitEvent(sc.fd, fb_merged[b], 0));
        CK(cudaMemcpyAsync(hacc_o + grow * BH * D, fb_o[b], size_t(n * BH * D * 4),
                           cudaMemcpyDeviceToHost, sc.fd));
        CK(cudaMemcpyAsync(hacc_l + grow * BH, fb_l[b], size_t(n * BH * 4), cudaMemcpyDeviceToHost,
                           sc.fd));
        CK(cudaEventRecord(fb_free[b], sc.fd));
        d2h += uint64_t(n * BH * (D + 1) * 4);
      }
    }
    ++gidx;
    if (j > 0) {
      CK(cudaEventRecord(flush_done, sc.fd));
      flushed_once = true;
    }
    gi = ge;
  }

  if (j > 0 && !direct_final) {  // host accumulator -> O, lse (after every flush): in = fb 0, out = fb 1
    CK(cudaEventRecord(flush_done, sc.fd));
    CK(cudaStreamWaitEvent(sc.fh, flush_done, 0));
    for (int64_t r = 0; r < N; r += F) {
      const int64_t n = std::min(F, N - r);
      CK(cudaStreamWaitEvent(sc.fh, fb_free[0], 0));   // (never-recorded events are no-ops)
      CK(cudaMemcpyAsync(fb_o[0], hacc_o + r * BH * D, size_t(n * BH * D * 4),
                         cudaMemcpyHostToDevice, sc.fh));
      CK(cudaMemcpyAsync(fb_l[0], hacc_l + r * BH, size_t(n * BH * 4), cudaMemcpyHostToDevice, sc.fh));
      CK(cudaEventRecord(fb_loaded[0], sc.fh));
      CK(cudaStreamWaitEvent(st, fb_loaded[0], 0));
      CK(cudaStreamWaitEvent(st, fb_free[1], 0));
      h2d += uint64_t(n * BH * (D + 1) * 4);
      cqs_status s2 = emit_final(1, fb_o[0], fb_l[0], r, n);
      if (s2 != CQS_OK) return s2;
      CK(cudaEventRecord(fb_free[0], st));   // input consumed by the kernel
    }
  }
  // the caller's stream must cover every copy issued on the helper streams
  CK(cudaEventRecord(flush_done, sc.fd));
  CK(cudaStreamWaitEvent(st, flush_done, 0));
  CK(cudaEventRecord(flush_done, sc.fh));
  CK(cudaStreamWaitEvent(st, flush_done, 0));

  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    CK(cudaStreamSynchronize(st));
    stats->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    stats->bytes_h2d = h2d;
    stats->bytes_d2h = d2h;
    stats->tasks_run = run;
    stats->tasks_skipped = int64_t(p->tasks.size()) - run;
    stats->kernel_launches = launches;
    stats->predicted_peak_bytes = p->predicted_peak;
  }
  (void)out_strides;
  return CQS_OK;
}

}  // namespace cqs

// CQS planner: Algorithm 3 BuildSubseq in segment form, the CQS mask
// (P:130-134), LPT task sharding and the device-memory model used to choose the
// divide depth from a byte budget (uniform scheduling; R14).
//
// Independent of oracle/: the oracle follows Alg. 3 literally on token arrays and dense masks; this
// planner never materialises token ids.  A leaf is a list of maximal *segments* (runs of
// consecutive global token ids whose per-level chunk codes are equal); the layout/gather steps of
// Alg. 3 are applied to segment lists, and the mask M_i is represented by the
// per-level codes: local pair (p,q) is masked iff at some level t both lie in the same non-owner
// chunk (code_t(p) == code_t(q) != 0), which is exactly "zero G x G for every group G" with the
// groups of P:295-298.  Every segment pair block is therefore wholly kept or wholly masked.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "cqs_internal.h"

namespace cqs {

static thread_local std::string g_err;

cqs_status fail(cqs_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }
// Bytes a device tensor of x bytes occupies in the caller's caching allocator (R14): below 1 MiB a
// 512-byte multiple carved from a shared small segment; from 1 MiB up its own segment of 2 MiB
// device pages (the driver's allocation granularity), so the allocator's view never exceeds it and
// a separately allocated tensor costs exactly this much free device memory.
uint64_t alloc_bytes(uint64_t x) {
  if (x < (uint64_t(1) << 20)) return (x + 511) & ~uint64_t(511);
  return (x + (uint64_t(2) << 20) - 1) & ~((uint64_t(2) << 20) - 1);
}

static int64_t elem_size(cqs_dtype t) { return t == CQS_BF16 ? 2 : 4; }

WsLayout ws_layout(const cqs_plan_desc& d, int64_t staged_rows, int64_t acc_rows,
                   int32_t n_stage_buffers) {
  const uint64_t BH = uint64_t(d.B) * d.H, D = d.D;
  WsLayout w{};
  uint64_t off = 0;
  w.acc_o = off;
  off += align256(uint64_t(acc_rows) * BH * D * 4);
  w.acc_lse = off;
  off += align256(uint64_t(acc_rows) * BH * 4);
  w.stage = off;
  w.stage_bytes_per_buf = 0;
  if (d.qkv_loc == CQS_LOC_PINNED_HOST) {
    // three tensors [BH][staged_rows][D] per buffer
    w.stage_bytes_per_buf = 3 * align256(BH * uint64_t(staged_rows) * D * elem_size(d.in_dtype));
    off += uint64_t(n_stage_buffers) * w.stage_bytes_per_buf;
  }
  w.flush = off;
  // flush buffers stage host-tier accumulator chunks and final rows (world = 1 streamed / host
  // output); a world > 1 call leaves its partials on the device for the exchange
  if (d.world == 1 && (d.qkv_loc == CQS_LOC_PINNED_HOST || d.out_loc == CQS_LOC_PINNED_HOST)) {
    const uint64_t F = uint64_t(flush_rows(acc_rows, int64_t(BH), int64_t(D)));
    off += 2 * (align256(F * BH * D * 4) + align256(F * BH * 4));
  }
  // n_parallel > 1 (resident): accumulator slots 1..P-1 for concurrently running tasks
  w.slots = off;
  w.slot_bytes = align256(uint64_t(acc_rows) * BH * D * 4) + align256(uint64_t(acc_rows) * BH * 4);
  if (d.qkv_loc == CQS_LOC_DEVICE && d.n_parallel > 1)
    off += uint64_t(d.n_parallel - 1) * w.slot_bytes;
  w.total = off;
  return w;
}

MemModel memory_model(const cqs_plan_desc& d, int64_t staged_rows, int64_t acc_rows,
                      int32_t n_stage_buffers, int64_t out_rows) {
  const uint64_t BH = uint64_t(d.B) * d.H, N = d.N, D = d.D, R = uint64_t(out_rows);
  MemModel m{};
  // every tensor counted as the caller's allocator holds it (alloc_bytes, R14): Q, K, V, O, lse
  // and the workspace allocated as separate tensors never occupy more than this
  m.caller_dev = 0;
  if (d.qkv_loc == CQS_LOC_DEVICE) m.caller_dev += 3 * alloc_bytes(BH * N * D * elem_size(d.in_dtype));
  if (d.out_loc == CQS_LOC_DEVICE || d.world > 1)
    m.caller_dev += alloc_bytes(BH * R * D * elem_size(d.out_dtype)) + alloc_bytes(4 * BH * R);
  m.dev_ws = alloc_bytes(ws_layout(d, staged_rows, acc_rows, n_stage_buffers).total);
  // pinned host accumulator of the host tier (world = 1 streamed plans with j > 0)
  m.host_ws = (d.world == 1 && acc_rows < d.N) ? align256(N * BH * D * 4) + align256(N * BH * 4) : 0;
  return m;
}

// ----- Algorithm 3 on segment lists ----------------------------------------------------------

// Chunk u of a length-L sequence: the first (L mod c) chunks get ceil(L/c) tokens (R1).
static inline void chunk_bounds(int64_t L, int c, int u, int64_t* a, int64_t* b) {
  const int64_t q = L / c, r = L % c;
  *a = u * q + std::min<int64_t>(u, r);
  *b = *a + q + (u < r ? 1 : 0);
}

// Segments of the depth-`depth` subsequence selected by quorum[0..depth).
// Returns false if more than CQS_MAX_SEGS segments arise.
bool build_segments(int64_t N, const Levels& lv, const int32_t* quorum, int depth,
                    std::vector<Seg>& out) {
  std::vector<Seg> cur(1), nxt;
  cur[0].start = 0;
  cur[0].len = N;
  std::memset(cur[0].codes, 0, sizeof(cur[0].codes));
  for (int t = 0; t < depth; ++t) {
    const int c = lv.c_at(t);
    const std::vector<int32_t>& I = lv.I_at(t);
    int64_t L = 0;
    for (auto& s : cur) L += s.len;
    nxt.clear();
    for (size_t i = 0; i < I.size(); ++i) {              // chunks in I order (R2)
      const int u = (quorum[t] + I[i]) % c;
      int64_t a, b;
      chunk_bounds(L, c, u, &a, &b);
      int64_t pos = 0;
      for (auto& s : cur) {                                // gather
        const int64_t lo = std::max(a, pos), hi = std::min(b, pos + s.len);
        if (lo < hi) {
          Seg p = s;
          p.start = s.start + (lo - pos);
          p.len = hi - lo;
          p.codes[t] = uint8_t(i);                         // label of this level
          if (!nxt.empty()) {
            Seg& q = nxt.back();
            if (q.start + q.len == p.start && std::memcmp(q.codes, p.codes, t + 1) == 0) {
              q.len += p.len;
              pos += s.len;
              continue;
            }
          }
          nxt.push_back(p);
        }
        pos += s.len;
      }
    }
    cur.swap(nxt);
    if (cur.size() > CQS_MAX_SEGS) return false;
  }
  out = cur;
  return true;
}

// Segment-block form of LocalMaskFromGroupRuns: masked iff some level puts both
// segments in the same non-owner chunk.
static inline bool kept_pair(const Seg& a, const Seg& b, int depth) {
  for (int t = 0; t < depth; ++t)
    if (a.codes[t] == b.codes[t] && a.codes[t] != 0) return false;
  return true;
}

static bool is_difference_set(const std::vector<int32_t>& I, int c) {
  std::vector<int> cnt(c, 0);
  for (size_t i = 0; i < I.size(); ++i)
    for (size_t j = 0; j < I.size(); ++j)
      if (i != j) cnt[((I[i] - I[j]) % c + c) % c]++;
  if (cnt[0] != 0) return false;
  for (int r = 1; r < c; ++r)
    if (cnt[r] != 1) return false;
  return true;
}

// Plan tables hold every task (~200 B each): cap the tree at 7^8 = 5.8M leaves.
constexpr int64_t kMaxTasks = 5764801;

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

// Longest depth-j subsequence (rows of one accumulator subtree) — lengths only.
static int64_t max_node_rows(int64_t N, const Levels& lv, int j) {
  std::vector<int64_t> lens{N}, nxt;
  for (int t = 0; t < j; ++t) {
    const int c = lv.c_at(t);
    const std::vector<int32_t>& I = lv.I_at(t);
    nxt.clear();
    std::vector<int64_t> uniq(lens);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    for (int64_t L : uniq)
      for (int q = 0; q < c; ++q) {
        int64_t tot = 0;
        for (int32_t o : I) {
          int64_t a, b;
          chunk_bounds(L, c, (q + o) % c, &a, &b);
          tot += b - a;
        }
        nxt.push_back(tot);
      }
    lens.swap(nxt);
  }
  return *std::max_element(lens.begin(), lens.end());
}

struct LeafSet {
  std::vector<Task> tasks;
  std::vector<Seg> segs;
  int64_t n_empty = 0, max_rows = 0, max_staged = 0;
  uint64_t total_work = 0;
};

// One leaf: segments of the subsequence at path quorum[0..depth), its kept segment-pair blocks,
// exact work and staged rows (segments touched by a kept block).
static cqs_status make_leaf(const cqs_plan_desc& d, const Levels& lv,
                            const int32_t* quorum, int depth, Task& T, std::vector<Seg>& segs,
                            int64_t* rows_out, int64_t* staged_out) {
  if (!build_segments(d.N, lv, quorum, depth, segs))
    return fail(CQS_E_UNSUPPORTED, "task has more than CQS_MAX_SEGS segments");
  T = Task{};
  T.depth = depth;
  std::copy(quorum, quorum + depth, T.quorum);
  T.nseg = int32_t(segs.size());
  uint32_t used = 0;
  int64_t rows = 0;
  for (int a = 0; a < T.nseg; ++a) {
    rows += segs[a].len;
    for (int b = 0; b < T.nseg; ++b)
      if (kept_pair(segs[a], segs[b], depth)) {
        T.kept[a] |= 1u << b;
        T.work += uint64_t(segs[a].len) * uint64_t(segs[b].len);
        used |= (1u << a) | (1u << b);
      }
  }
  int64_t staged = 0;
  for (int a = 0; a < T.nseg; ++a)
    if (used & (1u << a)) staged += segs[a].len;
  *rows_out = rows;
  *staged_out = staged;
  return CQS_OK;
}

static void add_leaf(LeafSet& ls, Task& T, const std::vector<Seg>& segs, int64_t rows,
                     int64_t staged) {
  T.seg_off = int64_t(ls.segs.size());
  ls.segs.insert(ls.segs.end(), segs.begin(), segs.end());
  ls.total_work += T.work;
  if (T.work == 0) ls.n_empty++;
  ls.max_rows = std::max(ls.max_rows, rows);
  ls.max_staged = std::max(ls.max_staged, staged);
  ls.tasks.push_back(T);
}

static cqs_status enumerate_leaves(const cqs_plan_desc& d, const Levels& lv, int depth,
                                   LeafSet& ls) {
  const int64_t n = lv.tasks(depth);
  ls = LeafSet{};
  ls.tasks.reserve(size_t(n));
  ls.segs.reserve(size_t(n) * 4);
  std::vector<Seg> segs;
  int32_t qt[CQS_MAX_DEPTH] = {};
  Task T;
  for (int64_t idx = 0; idx < n; ++idx) {
    int64_t r = idx;                                       // lexicographic, q_1 most significant
    for (int t = depth - 1; t >= 0; --t) {                 // (mixed radix for per-level c)
      qt[t] = int32_t(r % lv.c_at(t));
      r /= lv.c_at(t);
    }
    int64_t rows, staged;
    cqs_status st = make_leaf(d, lv, qt, depth, T, segs, &rows, &staged);
    if (st != CQS_OK) return st;
    add_leaf(ls, T, segs, rows, staged);
  }
  return CQS_OK;
}

// LPT on exact work (largest first, ties by index) -> least-loaded rank (ties lowest rank).
// Writes Task::rank; returns the makespan.
static uint64_t lpt_assign(std::vector<Task>& tasks, int world) {
  std::vector<int64_t> order;
  for (int64_t i = 0; i < int64_t(tasks.size()); ++i) {
    tasks[size_t(i)].rank = -1;
    if (tasks[size_t(i)].work > 0) order.push_back(i);
  }
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return tasks[size_t(a)].work > tasks[size_t(b)].work;
  });
  std::vector<uint64_t> load(size_t(world), 0);
  for (int64_t i : order) {
    const size_t r = size_t(std::min_element(load.begin(), load.end()) - load.begin());
    tasks[size_t(i)].rank = int32_t(r);
    load[r] += tasks[size_t(i)].work;
  }
  return *std::max_element(load.begin(), load.end());
}

// Contiguous assignment: non-empty tasks in lexicographic (DFS) order; a task goes to the rank
// whose equal-work interval contains the midpoint of its work on the prefix-sum axis, so rank r
// takes one consecutive run of tasks (a few neighbouring subtrees).  Returns the makespan.
static uint64_t contiguous_assign(std::vector<Task>& tasks, int world) {
  uint64_t total = 0;
  for (const Task& T : tasks) total += T.work;
  std::vector<uint64_t> load(size_t(world), 0);
  uint64_t pre = 0;
  for (Task& T : tasks) {
    T.rank = -1;
    if (T.work == 0) continue;
    const long double mid = (long double)pre + (long double)T.work / 2;
    int r = int(mid * world / (long double)total);
    r = std::min(std::max(r, 0), world - 1);
    T.rank = r;
    load[size_t(r)] += T.work;
    pre += T.work;
  }
  return *std::max_element(load.begin(), load.end());
}

static uint64_t assign_ranks(std::vector<Task>& tasks, const cqs_plan_desc& d) {
  if (d.world > 1 && d.shard == CQS_SHARD_CONTIGUOUS) return contiguous_assign(tasks, d.world);
  return lpt_assign(tasks, d.world);
}

void held_blocks(const std::vector<Task>& tasks, const std::vector<Seg>& segs, int64_t N,
                 int32_t r, std::vector<uint8_t>& held) {
  const int64_t G = CQS_ACC_BLOCK_ROWS;
  held.assign(size_t((N + G - 1) / G), 0);
  for (const Task& T : tasks) {
    if (T.rank != r) continue;
    for (int a = 0; a < T.nseg; ++a) {
      if (!T.kept[a]) continue;                          // not an active query segment
      const Seg& sg = segs[size_t(T.seg_off + a)];
      for (int64_t b = sg.start / G; b <= (sg.start + sg.len - 1) / G; ++b) held[size_t(b)] = 1;
    }
  }
}

// Accumulator rows every rank needs (world > 1): held blocks x CQS_ACC_BLOCK_ROWS.
static std::vector<int64_t> held_rows_per_rank(const std::vector<Task>& tasks,
                                               const std::vector<Seg>& segs, int64_t N,
                                               int world) {
  const int64_t G = CQS_ACC_BLOCK_ROWS, nb = (N + G - 1) / G;
  std::vector<uint8_t> held(size_t(nb) * size_t(world), 0);
  for (const Task& T : tasks) {
    if (T.rank < 0) continue;
    uint8_t* h = held.data() + size_t(T.rank) * size_t(nb);
    for (int a = 0; a < T.nseg; ++a) {
      if (!T.kept[a]) continue;
      const Seg& sg = segs[size_t(T.seg_off + a)];
      for (int64_t b = sg.start / G; b <= (sg.start + sg.len - 1) / G; ++b) h[b] = 1;
    }
  }
  std::vector<int64_t> rows(size_t(world), 0);
  for (int r = 0; r < world; ++r) {
    int64_t c = 0;
    for (int64_t b = 0; b < nb; ++b) c += held[size_t(r) * size_t(nb) + size_t(b)];
    rows[size_t(r)] = c * G;
  }
  return rows;
}

static int64_t shard_rows_of(int64_t N, int world, int rank) {
  return (N * (rank + 1)) / world - (N * rank) / world;
}

// Hybrid scheduling (Fig. "schedule" right): leaves at mixed depths.  Starting from the
// uniform tree, repeatedly replace the heaviest leaf (ties: first in DFS order) by its c children
// until the LPT makespan is within 1% of total/world.  Any such tree is still an exact
// decomposition: a node's c children partition its kept pairs (the per-level invariant of CQS
// Divide), so every ordered pair stays covered exactly once.
constexpr int64_t kMaxHybridLeaves = 4096;
static cqs_status refine_hybrid(const cqs_plan_desc& d, const Levels& lv, LeafSet& ls) {
  struct Leaf {
    Task T;
    std::vector<Seg> segs;
    int64_t rows, staged;
  };
  std::vector<Leaf> leaves(ls.tasks.size());
  for (size_t i = 0; i < ls.tasks.size(); ++i) {
    const Task& T = ls.tasks[i];
    leaves[i].T = T;
    leaves[i].segs.assign(ls.segs.begin() + T.seg_off, ls.segs.begin() + T.seg_off + T.nseg);
    int64_t rows = 0;
    for (auto& sg : leaves[i].segs) rows += sg.len;
    leaves[i].rows = rows;
    leaves[i].staged = rows;
  }
  const uint64_t total = ls.total_work;
  for (;;) {
    std::vector<Task> ts;
    for (auto& L : leaves) ts.push_back(L.T);
    const uint64_t span = lpt_assign(ts, d.world);
    if (double(span) <= 1.01 * double(total) / d.world) break;
    size_t best = 0;
    for (size_t i = 1; i < leaves.size(); ++i)
      if (leaves[i].T.work > leaves[best].T.work) best = i;
    const Task P = leaves[best].T;
    const int ck = lv.c_at(P.depth);                      // children of a depth-t node: c_t
    if (int64_t(leaves.size()) + ck - 1 > kMaxHybridLeaves) break;
    if (P.depth + 1 >= CQS_MAX_DEPTH) break;
    // children need at least one token per chunk of the parent's length
    if (leaves[best].rows < ck) break;
    std::vector<Leaf> kids(static_cast<size_t>(ck));
    int32_t qt[CQS_MAX_DEPTH] = {};
    std::copy(P.quorum, P.quorum + P.depth, qt);
    for (int q = 0; q < ck; ++q) {
      qt[P.depth] = q;
      cqs_status st = make_leaf(d, lv, qt, P.depth + 1, kids[size_t(q)].T, kids[size_t(q)].segs,
                                &kids[size_t(q)].rows, &kids[size_t(q)].staged);
      if (st != CQS_OK) return st;
    }
    leaves.erase(leaves.begin() + long(best));
    leaves.insert(leaves.begin() + long(best), kids.begin(), kids.end());
  }
  LeafSet out;
  for (auto& L : leaves) add_leaf(out, L.T, L.segs, L.rows, L.staged);
  ls = std::move(out);
  return CQS_OK;
}

}  // namespace cqs

using namespace cqs;

extern "C" {

const char* cqs_last_error(void) { return g_err.c_str(); }
int32_t cqs_abi_version(void) { return CQS_ABI_VERSION; }

// One interest set: c = l(l-1)+1, offsets distinct in [0, c), offsets[0] = 0 (R4), and a
// (c, l, 1) difference set.
static cqs_status check_set(int c, int l, const int32_t* offs, std::vector<int32_t>& I) {
  if (l < 1 || c != l * (l - 1) + 1) return fail(CQS_E_INVALID, "c must equal l(l-1)+1 (P:30)");
  if (!offs) return fail(CQS_E_INVALID, "offsets is NULL");
  I.assign(offs, offs + l);
  for (int i = 0; i < l; ++i) {
    if (I[i] < 0 || I[i] >= c) return fail(CQS_E_INVALID, "offset out of [0, c)");
    for (int j = 0; j < i; ++j)
      if (I[i] == I[j]) return fail(CQS_E_INVALID, "duplicate offset");
  }
  if (I[0] != 0) return fail(CQS_E_INVALID, "offsets[0] must be 0 (owner chunk, R4)");
  if (!is_difference_set(I, c))
    return fail(CQS_E_INVALID, "interest set is not a (c,l,1) difference set (P:352)");
  return CQS_OK;
}

static int l_of_c(int c) {   // l with l(l-1)+1 = c, or 0
  for (int l = 1; l * (l - 1) + 1 <= c; ++l)
    if (l * (l - 1) + 1 == c) return l;
  return 0;
}

static cqs_status validate_desc(const cqs_plan_desc* d, Levels& lv) {
  if (!d) return fail(CQS_E_INVALID, "desc is NULL");
  if (d->N < 1 || d->N > INT32_MAX) return fail(CQS_E_INVALID, "N must be in [1, 2^31)");
  if (d->B < 1 || d->H < 1 || d->D < 1) return fail(CQS_E_INVALID, "B, H, D must be >= 1");
  lv = Levels{};
  lv.c = d->c;
  cqs_status st = check_set(d->c, d->l, d->offsets, lv.I);
  if (st != CQS_OK) return st;
  if (d->n_level_sets < 0 || d->n_level_sets > CQS_MAX_DEPTH)
    return fail(CQS_E_INVALID, "n_level_sets out of [0, CQS_MAX_DEPTH]");
  if (d->n_level_sets > 0 && (!d->level_c || !d->level_offsets))
    return fail(CQS_E_INVALID, "level_c / level_offsets NULL");
  for (int t = 0, o = 0; t < d->n_level_sets; ++t) {
    const int c = d->level_c[t], l = l_of_c(c);
    if (l == 0) return fail(CQS_E_INVALID, "level c must be l(l-1)+1 (P:30)");
    std::vector<int32_t> I;
    if ((st = check_set(c, l, d->level_offsets + o, I)) != CQS_OK) return st;
    lv.lc.push_back(c);
    lv.lI.push_back(I);
    o += l;
  }
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world)
    return fail(CQS_E_INVALID, "bad world/rank");
  if (d->depth < -1 || d->depth >= CQS_MAX_DEPTH) return fail(CQS_E_INVALID, "bad depth");
  if (d->depth >= 0 && d->N < lv.tasks(d->depth))
    return fail(CQS_E_INVALID, "N < c^depth (R10; product of the level c's for mixed trees)");
  if (d->depth >= 0 && lv.tasks(d->depth) > kMaxTasks)
    return fail(CQS_E_UNSUPPORTED, "more than 7^8 tasks: the plan table would not fit host memory");
  if (d->in_dtype == CQS_BF16 && !(d->D == 64 || d->D == 128))
    return fail(CQS_E_UNSUPPORTED, "bf16 path supports D in {64, 128}");
  if (d->in_dtype == CQS_F32 && !(d->D % 32 == 0 && d->D <= 128))
    return fail(CQS_E_UNSUPPORTED, "fp32 path supports D in {32, 64, 96, 128}");
  if (d->qkv_loc == CQS_LOC_DEVICE && d->out_loc != CQS_LOC_DEVICE)
    return fail(CQS_E_UNSUPPORTED, "resident Q/K/V require a device output");
  if (d->schedule != CQS_SCHED_UNIFORM && d->schedule != CQS_SCHED_HYBRID)
    return fail(CQS_E_INVALID, "schedule must be CQS_SCHED_UNIFORM or CQS_SCHED_HYBRID");
  if (d->shard != CQS_SHARD_LPT && d->shard != CQS_SHARD_CONTIGUOUS)
    return fail(CQS_E_INVALID, "shard must be CQS_SHARD_LPT or CQS_SHARD_CONTIGUOUS");
  if (d->flags & ~CQS_PLAN_SUBSET) return fail(CQS_E_INVALID, "unknown flags");
  if (d->reserved1 != 0) return fail(CQS_E_INVALID, "reserved1 must be 0");
  if (d->n_parallel < 0 || d->n_parallel > 8) return fail(CQS_E_INVALID, "n_parallel in [0, 8]");
  if (d->n_parallel > 1 && d->qkv_loc != CQS_LOC_DEVICE)
    return fail(CQS_E_UNSUPPORTED, "n_parallel > 1: resident plans only (the streamed executor "
                                   "overlaps staging with one task at a time)");
  if ((d->flags & CQS_PLAN_SUBSET) && !d->exec_order)
    return fail(CQS_E_INVALID, "CQS_PLAN_SUBSET needs exec_order");
  if (d->n_exec_order < 0 || (d->n_exec_order > 0 && !d->exec_order))
    return fail(CQS_E_INVALID, "exec_order NULL with n_exec_order > 0");
  if (d->schedule == CQS_SCHED_HYBRID && d->qkv_loc == CQS_LOC_PINNED_HOST)
    return fail(CQS_E_UNSUPPORTED, "hybrid schedule: resident plans only (the streamed executor "
                                   "groups uniform subtrees)");
  return CQS_OK;
}

// Device bytes of a world > 1 call at this leaf set: the task assignment decides each rank's
// accumulator rows (held blocks); `mine` = this rank's model, return value = the largest over the
// ranks (the depth / buffer choice must be the same on every rank, and every rank must fit).
static MemModel sharded_model(const cqs_plan_desc& d, LeafSet& ls, int64_t staged, int nbuf,
                              MemModel* mine, int64_t* my_acc_rows) {
  assign_ranks(ls.tasks, d);
  const std::vector<int64_t> rows = held_rows_per_rank(ls.tasks, ls.segs, d.N, d.world);
  MemModel worst{};
  for (int r = 0; r < d.world; ++r) {
    MemModel m = memory_model(d, staged, rows[size_t(r)], nbuf, shard_rows_of(d.N, d.world, r));
    if (m.caller_dev + m.dev_ws > worst.caller_dev + worst.dev_ws) worst = m;
    if (r == d.rank) *mine = m, *my_acc_rows = rows[size_t(r)];
  }
  return worst;
}

cqs_status cqs_memory_model(const cqs_plan_desc* desc, int32_t depth, int32_t acc_depth,
                            int32_t n_stage_buffers, uint64_t* dev_bytes, uint64_t* host_bytes) {
  Levels lv;
  cqs_status st = validate_desc(desc, lv);
  if (st != CQS_OK) return st;
  if (depth < 0 || depth >= CQS_MAX_DEPTH || acc_depth < 0 || acc_depth > depth ||
      desc->N < lv.tasks(depth))
    return fail(CQS_E_INVALID, "bad depth / acc_depth");
  const bool streamed = desc->qkv_loc == CQS_LOC_PINNED_HOST, sharded = desc->world > 1;
  if (sharded && acc_depth != 0)
    return fail(CQS_E_INVALID, "world > 1 keeps a device accumulator (acc_depth 0)");
  LeafSet ls;
  int64_t staged = desc->N;
  if (streamed || sharded) {
    if ((st = enumerate_leaves(*desc, lv, depth, ls)) != CQS_OK) return st;
    staged = ls.max_staged;
  }
  MemModel m;
  if (sharded) {
    MemModel mine{};
    int64_t rows = 0;
    m = sharded_model(*desc, ls, streamed ? staged : 0, streamed ? n_stage_buffers : 0, &mine,
                      &rows);
    m = mine;   // this rank's bytes (cqs_plan chooses by the largest over the ranks)
  } else {
    const int64_t acc_rows = streamed ? max_node_rows(desc->N, lv, acc_depth) : desc->N;
    m = memory_model(*desc, streamed ? staged : 0, acc_rows, streamed ? n_stage_buffers : 0,
                     desc->N);
  }
  if (dev_bytes) *dev_bytes = m.caller_dev + m.dev_ws;
  if (host_bytes) *host_bytes = m.host_ws;
  return CQS_OK;
}

cqs_status cqs_plan(const cqs_plan_desc* desc, cqs_plan_t** out) {
  if (!out) return fail(CQS_E_INVALID, "out is NULL");
  *out = nullptr;
  Levels lv;
  cqs_status st = validate_desc(desc, lv);
  if (st != CQS_OK) return st;
  const cqs_plan_desc& d = *desc;
  const bool streamed = d.qkv_loc == CQS_LOC_PINNED_HOST, sharded = d.world > 1;
  const uint64_t budget = d.budget_bytes;

  int max_depth = 0;
  while (max_depth + 1 < CQS_MAX_DEPTH && lv.tasks(max_depth + 1) <= d.N &&
         lv.tasks(max_depth + 1) <= kMaxTasks)
    ++max_depth;
  const int k_lo = d.depth >= 0 ? d.depth : 0, k_hi = d.depth >= 0 ? d.depth : max_depth;

  LeafSet ls;
  int chosen = -1, chosen_j = 0, chosen_nbuf = 0;
  int64_t acc_rows = d.N;
  MemModel mm{};
  auto fits = [&](const MemModel& m) { return budget == 0 || m.caller_dev + m.dev_ws <= budget; };
  if (!streamed && !sharded) {
    // resident single-GPU bytes do not depend on the depth: decide feasibility once, then
    // enumerate only the chosen depth (the smallest one, or the caller's)
    mm = memory_model(d, 0, d.N, 0, d.N);
    if (!fits(mm))
      return fail(CQS_E_INFEASIBLE, "resident plan exceeds budget_bytes at every depth");
    if ((st = enumerate_leaves(d, lv, k_lo, ls)) != CQS_OK) return st;
    chosen = k_lo;
  }
  for (int k = k_lo; k <= k_hi && chosen < 0; ++k) {
    if ((st = enumerate_leaves(d, lv, k, ls)) != CQS_OK) return st;
    if (sharded) {
      // rank-local accumulators (held blocks) on the device; streamed: plus staging buffers
      for (int nbuf = streamed ? 2 : 0; nbuf >= (streamed ? 1 : 0) && chosen < 0; --nbuf) {
        MemModel mine{};
        int64_t rows = 0;
        const MemModel worst = sharded_model(d, ls, streamed ? ls.max_staged : 0, nbuf, &mine, &rows);
        if (fits(worst)) chosen = k, chosen_j = 0, chosen_nbuf = nbuf, acc_rows = rows, mm = mine;
      }
      continue;
    }
    for (int nbuf = 2; nbuf >= 1 && chosen < 0; --nbuf)
      for (int j = 0; j <= k && chosen < 0; ++j) {
        const int64_t rows = max_node_rows(d.N, lv, j);
        MemModel m = memory_model(d, ls.max_staged, rows, nbuf, d.N);
        if (fits(m)) chosen = k, chosen_j = j, chosen_nbuf = nbuf, acc_rows = rows, mm = m;
      }
  }
  if (chosen < 0)
    return fail(CQS_E_INFEASIBLE, "no divide depth fits budget_bytes under the memory model");
  if (d.schedule == CQS_SCHED_HYBRID && d.world > 1)
    if ((st = refine_hybrid(d, lv, ls)) != CQS_OK) return st;

  auto* p = new cqs_plan_t();
  p->desc = d;
  p->lv = lv;
  p->desc.offsets = p->lv.I.data();
  // the plan owns its level tables (the caller's arrays may go away)
  for (auto& I : p->lv.lI) p->level_offsets.insert(p->level_offsets.end(), I.begin(), I.end());
  p->desc.level_c = p->lv.lc.empty() ? nullptr : p->lv.lc.data();
  p->desc.level_offsets = p->level_offsets.empty() ? nullptr : p->level_offsets.data();
  p->desc.exec_order = nullptr;
  p->desc.n_exec_order = 0;
  p->depth = chosen;
  p->max_depth = chosen;
  for (const Task& T : ls.tasks) p->max_depth = std::max(p->max_depth, T.depth);
  p->acc_depth = streamed ? chosen_j : 0;
  p->n_stage_buffers = streamed ? chosen_nbuf : 0;
  p->tasks.swap(ls.tasks);
  p->segs.swap(ls.segs);
  p->n_empty = ls.n_empty;
  p->max_task_rows = ls.max_rows;
  p->max_staged_rows = streamed ? ls.max_staged : 0;
  p->total_work = ls.total_work;

  assign_ranks(p->tasks, d);
  for (int64_t i = 0; i < int64_t(p->tasks.size()); ++i)
    if (p->tasks[size_t(i)].rank == d.rank) {
      p->my_order.push_back(i);
      p->my_work += p->tasks[size_t(i)].work;
    }
  if (d.exec_order) {   // caller's execution order (any order is exact, Eq. 3) or subset
    const int64_t n = int64_t(p->tasks.size());
    const bool subset = d.flags & CQS_PLAN_SUBSET;
    if (!subset && d.n_exec_order != n) {
      delete p;
      return fail(CQS_E_INVALID, "exec_order must list all " + std::to_string(n) + " tasks");
    }
    std::vector<int64_t> pos(size_t(n), -1);
    for (int64_t i = 0; i < d.n_exec_order; ++i) {
      const int64_t t = d.exec_order[i];
      if (t < 0 || t >= n || pos[size_t(t)] >= 0) {
        delete p;
        return fail(CQS_E_INVALID, "exec_order entries must be distinct task indices");
      }
      pos[size_t(t)] = i;
    }
    if (subset) {   // only the listed tasks of this rank, in the listed order
      std::vector<int64_t> mine;
      p->my_work = 0;
      for (int64_t i = 0; i < d.n_exec_order; ++i) {
        const Task& T = p->tasks[size_t(d.exec_order[i])];
        if (T.rank == d.rank && T.work > 0) {
          mine.push_back(d.exec_order[i]);
          p->my_work += T.work;
        }
      }
      p->my_order.swap(mine);
    } else {
      std::stable_sort(p->my_order.begin(), p->my_order.end(),
                       [&](int64_t a, int64_t b) { return pos[size_t(a)] < pos[size_t(b)]; });
    }
  }
  if (sharded) {
    // rank-local accumulator: held blocks packed in increasing global order
    std::vector<uint8_t> held;
    held_blocks(p->tasks, p->segs, d.N, d.rank, held);
    p->acc_slot.assign(held.size(), -1);
    int32_t nb = 0;
    for (size_t b = 0; b < held.size(); ++b)
      if (held[b]) p->acc_slot[b] = nb++;
    acc_rows = int64_t(nb) * CQS_ACC_BLOCK_ROWS;
    p->shard_rows = shard_rows_of(d.N, d.world, d.rank);
    // (hybrid refinement may have changed the leaves: re-evaluate this rank's bytes)
    mm = memory_model(d, p->max_staged_rows, acc_rows, p->n_stage_buffers, p->shard_rows);
  }
  p->max_acc_rows = acc_rows;
  p->dev_ws = mm.dev_ws;
  p->host_ws = mm.host_ws;
  p->predicted_peak = mm.caller_dev + mm.dev_ws;
  *out = p;
  return CQS_OK;
}

cqs_status cqs_plan_info(const cqs_plan_t* p, cqs_plan_info_t* info) {
  if (!p || !info) return fail(CQS_E_INVALID, "NULL argument");
  std::memset(info, 0, sizeof(*info));
  info->depth = p->depth;
  info->acc_depth = p->acc_depth;
  info->n_stage_buffers = p->n_stage_buffers;
  info->max_depth = p->max_depth;
  info->n_tasks = int64_t(p->tasks.size());
  info->n_empty = p->n_empty;
  info->max_task_rows = p->max_task_rows;
  info->max_staged_rows = p->max_staged_rows;
  info->total_work_pairs = p->total_work;
  info->my_tasks = int64_t(p->my_order.size());
  info->my_work_pairs = p->my_work;
  info->dev_workspace_bytes = p->dev_ws;
  info->host_workspace_bytes = p->host_ws;
  info->predicted_peak_bytes = p->predicted_peak;
  info->acc_rows = p->max_acc_rows;
  info->shard_rows = p->desc.world > 1 ? p->shard_rows : 0;
  return CQS_OK;
}

cqs_status cqs_plan_task(const cqs_plan_t* p, int64_t idx, cqs_task_t* t) {
  if (!p || !t) return fail(CQS_E_INVALID, "NULL argument");
  if (idx < 0 || idx >= int64_t(p->tasks.size())) return fail(CQS_E_INVALID, "task index");
  std::memset(t, 0, sizeof(*t));
  const Task& T = p->tasks[size_t(idx)];
  t->nseg = T.nseg;
  t->rank = T.rank;
  t->depth = T.depth;
  t->work = T.work;
  std::copy(T.quorum, T.quorum + CQS_MAX_DEPTH, t->quorum);
  for (int a = 0; a < T.nseg; ++a) {
    const Seg& s = p->segs[size_t(T.seg_off + a)];
    t->seg_start[a] = s.start;
    t->seg_len[a] = s.len;
    std::memcpy(t->seg_codes[a], s.codes, CQS_MAX_DEPTH);
    t->kept[a] = T.kept[a];
  }
  return CQS_OK;
}

cqs_status cqs_plan_serialize(const cqs_plan_t* p, void* buf, size_t* len) {
  if (!p || !len) return fail(CQS_E_INVALID, "NULL argument");
  std::string b;
  auto put = [&](const void* x, size_t n) { b.append(static_cast<const char*>(x), n); };
  // v1: uniform tree; v2: hybrid (leaves of mixed depth); v3: per-level interest sets
  const bool mixed_depth = p->max_depth != p->depth, levels = p->lv.mixed();
  const uint32_t ver = levels ? 3 : (mixed_depth ? 2 : 1);
  const bool per_task_depth = ver >= 2;
  b.append("CQSP", 4);
  put(&ver, 4);
  put(&p->desc.N, 8);
  if (ver == 3) {
    put(&p->depth, 4);
    const int32_t nl = p->max_depth;          // the level table covers every leaf's levels
    put(&nl, 4);
    for (int t = 0; t < nl; ++t) {
      const int32_t c = p->lv.c_at(t), l = int32_t(p->lv.I_at(t).size());
      put(&c, 4);
      put(&l, 4);
      put(p->lv.I_at(t).data(), 4 * size_t(l));
    }
  } else {
    put(&p->desc.c, 4);
    put(&p->desc.l, 4);
    put(p->lv.I.data(), 4 * p->lv.I.size());
    put(&p->depth, 4);
  }
  const int64_t nt = int64_t(p->tasks.size());
  put(&nt, 8);
  for (const Task& T : p->tasks) {
    if (per_task_depth) put(&T.depth, 4);
    put(&T.nseg, 4);
    put(&T.work, 8);
    for (int a = 0; a < T.nseg; ++a) {
      const Seg& s = p->segs[size_t(T.seg_off + a)];
      put(&s.start, 8);
      put(&s.len, 8);
      put(s.codes, size_t(T.depth));
    }
    put(T.kept, 4 * size_t(T.nseg));
  }
  if (!buf) {
    *len = b.size();
    return CQS_OK;
  }
  if (*len < b.size()) {
    *len = b.size();
    return fail(CQS_E_INVALID, "buffer too small");
  }
  std::memcpy(buf, b.data(), b.size());
  *len = b.size();
  return CQS_OK;
}

void cqs_plan_destroy(cqs_plan_t* p) { delete p; }

cqs_status cqs_forward_workspace_size(const cqs_plan_t* p, size_t* dev_bytes, size_t* host_bytes) {
  if (!p) return fail(CQS_E_INVALID, "plan is NULL");
  if (dev_bytes) *dev_bytes = size_t(p->dev_ws);
  if (host_bytes) *host_bytes = size_t(p->host_ws);
  return CQS_OK;
}

cqs_status cqs_shard_rows(int64_t N, int32_t world, int32_t rank, int64_t* row0, int64_t* rows) {
  if (world < 1 || rank < 0 || rank >= world || N < 0 || !row0 || !rows)
    return fail(CQS_E_INVALID, "bad shard arguments");
  const int64_t a = (N * rank) / world, b = (N * (rank + 1)) / world;
  *row0 = a;
  *rows = b - a;
  return CQS_OK;
}

}  // extern "C"

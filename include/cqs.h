/*
 * cqs.h — C ABI of libcqs: exact softmax attention decomposed by CQS Divide (Stream-CQSA,
 * arXiv 2604.20819), B200 (sm_100a): forward hot path, backward (Algorithm 2), multi-GPU exchange.
 *
 * Citations: P:n = PAPER.md line n (section in brackets).  R<n> = DESIGN.md reading n.
 *
 * Problem statement (P:8 [Abstract], P:19 [Intro], P:60 [Alg. 1 Require], P:248 [Sec. 4]):
 *   given Q, K, V in R^{B x H x N x D} and a device-memory budget, return
 *   O = softmax(alpha Q K^T) V  (alpha = 1/sqrt(D), non-causal) computed as c^itr independent
 *   CQS tasks whose LSE-merge is exactly full attention.
 *
 * Conventions (all entry points):
 *   - Every tensor and workspace is owned by the caller; libcqs never allocates device or pinned
 *     memory and never frees caller memory.  Workspace sizes are queried up front.
 *   - Plans are immutable after cqs_plan() and may be shared between threads.
 *   - Device calls are asynchronous on `stream`; argument errors are detected on the host before
 *     any launch and reported synchronously.  CUDA launch/runtime errors map to CQS_E_CUDA.
 *   - On any non-OK status a thread-local message is available from cqs_last_error().
 *   - Determinism: a fixed plan (task order, merge order) gives bit-identical output across runs.
 */
#ifndef CQS_H_
#define CQS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CQS_ABI_VERSION 5
#define CQS_MAX_DEPTH 12   /* N >= 7^depth and N < 2^31 imply depth <= 11 for c = 7           */
#define CQS_MAX_SEGS 32    /* segments per task; observed <= 8 up to depth 11     */

typedef enum {
  CQS_OK = 0,
  CQS_E_VERIFY = 1,       /* internal consistency check failed                                 */
  CQS_E_INFEASIBLE = 2,   /* no depth fits budget_bytes (S:431 exit code 2)                    */
  CQS_E_INVALID = 3,      /* bad argument: I not a difference set, N < c^depth, ...    */
  CQS_E_CUDA = 4,         /* CUDA runtime / launch failure                                     */
  CQS_E_NCCL = 5,
  CQS_E_OOM = 6,          /* caller-provided workspace smaller than the queried size           */
  CQS_E_UNSUPPORTED = 7   /* valid request this build has no kernel for (dtype / D / segs)     */
} cqs_status;

typedef enum { CQS_F32 = 0, CQS_BF16 = 1 } cqs_dtype;
typedef enum { CQS_LOC_DEVICE = 0, CQS_LOC_PINNED_HOST = 1 } cqs_loc;

/* ---------------------------------------------------------------------------------------------
 * Planning (CQS Divide, Algorithm 3 BuildSubseq; masking P:130-134)
 * --------------------------------------------------------------------------------------------- */
typedef struct {
  int64_t N;                 /* tokens                                                        */
  int32_t B, H, D;           /* batch, heads, head dim; (b,h) planes are independent (R11)    */
  int32_t c, l;              /* chunk count c = l(l-1)+1                               */
  const int32_t* offsets;    /* interest set I, l entries, host memory, must be a (c,l,1)
                                difference set with offsets[0] == 0 (owner code 0, R4) */
  int32_t depth;             /* itr >= 0 explicit (0 = one task = plain attention); -1 = the
                                smallest depth whose predicted device bytes fit budget_bytes
                                (uniform scheduling; R14)                          */
  uint64_t budget_bytes;     /* device bytes the call may use incl. caller device tensors (R14);
                                0 = unlimited                                                  */
  cqs_dtype in_dtype;        /* Q, K, V element type: CQS_BF16 (tcgen05 path) or CQS_F32     */
  cqs_dtype out_dtype;       /* O element type                                                */
  cqs_loc qkv_loc;           /* where Q, K, V live: device (resident) or pinned host (stream) */
  cqs_loc out_loc;           /* where O and lse live                                          */
  int32_t world, rank;       /* task sharding across `world` GPUs; world=1 on 1 GPU */
  int32_t schedule;          /* CQS_SCHED_UNIFORM: every leaf at `depth`.  CQS_SCHED_HYBRID
                                (resident plans, P:158 hybrid scheduling): start from the uniform
                                tree and split the heaviest leaf into its c children until the LPT
                                makespan over `world` ranks is within 1% of work/world (or 4096
                                leaves); a no-op for world = 1.  Leaves then sit at mixed depths. */
  int32_t n_level_sets;      /* 0: every level uses (c, offsets).  k > 0: divide level t < k uses
                                interest set t below ("different values of c ... at each
                                iteration"), deeper levels (c, offsets).  Task count = product of
                                the levels' c; N must be >= that product (R10).               */
  const int32_t* level_c;    /* n_level_sets chunk counts, each l(l-1)+1                      */
  const int32_t* level_offsets; /* concatenated offsets, l_t per level, each a difference set
                                   with offsets[0] = 0 (host memory, copied by cqs_plan)    */
  int32_t shard;             /* world > 1 task assignment (tasks are independent, so
                                any assignment is exact).  CQS_SHARD_LPT: largest work first to
                                the least-loaded rank (best balance).  CQS_SHARD_CONTIGUOUS:
                                ranks take consecutive runs of the lexicographic (DFS) task order
                                split at equal work, so a rank's tasks share subtrees and touch
                                fewer rows — its accumulator (which holds only the rows its tasks
                                touch, see cqs_partial_runs) shrinks, e.g. to <= 70% of N at
                                C4 / world 8.  Ignored when world = 1.                          */
  int32_t flags;             /* CQS_PLAN_SUBSET: exec_order lists a SUBSET of the tasks (distinct
                                indices) and the call runs only those (of this rank), in that
                                order — the output then holds the LSE merge of their partials
                                only (rows they never touch: O = 0 and lse = -inf, or left
                                unwritten by the streamed executor with a host-tier
                                accumulator, which never reads or writes host rows outside the
                                listed tasks' subsequences).  For splitting
                                one tree over several calls / schedulers and for sampled
                                measurement (SURVEY §8d C5 protocol).  Other bits must be 0.   */
  const int64_t* exec_order; /* NULL, or a permutation of [0, n_tasks) (host memory, copied): the
                                rank runs its tasks in this relative order instead of the
                                lexicographic one.  Any order is exact (the LSE merge is
                                associative and commutative, Eq. 3) up to fp rounding.
                                CQS_E_INVALID if not a permutation of the planned task count
                                (without CQS_PLAN_SUBSET) or not distinct valid indices.        */
  int64_t n_exec_order;
  int32_t n_parallel;        /* tasks in flight ("n_parallel"): 0 or 1 = one task at a
                                time on the caller's stream; P in [2, 8] (resident plans) = this
                                rank's tasks round-robin over P streams, each with its own fp32
                                accumulator slot (the in-place merge of one slot is never shared
                                by concurrent tasks), merged into slot 0 at the end (Eq. 3).
                                Costs (P - 1) extra accumulators in the memory model; pays off
                                when single tasks do not fill the GPU (deep trees, few heads). */
  int32_t reserved1;         /* must be 0                                                       */
} cqs_plan_desc;

#define CQS_SCHED_UNIFORM 0
#define CQS_SCHED_HYBRID 1
#define CQS_SHARD_LPT 0
#define CQS_SHARD_CONTIGUOUS 1
#define CQS_PLAN_SUBSET 1
/* Rank-local accumulators (world > 1) are kept in blocks of this many consecutive rows. */
#define CQS_ACC_BLOCK_ROWS 256

typedef struct cqs_plan_s cqs_plan_t; /* opaque, library-owned, immutable */

typedef struct {
  int32_t depth;                 /* itr actually planned                                       */
  int32_t acc_depth;             /* device accumulator tier: rows of one depth-j subtree (0=all N) */
  int32_t n_stage_buffers;       /* streamed mode: staging buffers (1 or 2), 0 when resident   */
  int32_t max_depth;             /* deepest leaf (= depth for uniform plans)                   */
  int64_t n_tasks;               /* c^depth                                            */
  int64_t n_empty;               /* tasks with no kept pair (never launched, R9)               */
  int64_t max_task_rows;         /* longest leaf                                               */
  int64_t max_staged_rows;       /* most rows any task stages (streamed mode)                  */
  uint64_t total_work_pairs;     /* sum of kept (q,k) pairs over all tasks = N^2 exactly       */
  int64_t my_tasks;              /* non-empty tasks assigned to `rank` (LPT on work)           */
  uint64_t my_work_pairs;
  uint64_t dev_workspace_bytes;  /* = cqs_forward_workspace_size(...).dev                      */
  uint64_t host_workspace_bytes; /* pinned host bytes (streamed mode)                          */
  uint64_t predicted_peak_bytes; /* memory model M_dev: caller device tensors + dev workspace
                                    (each tensor at the allocator's 512-byte granularity, R14);
                                    world > 1: this rank's bytes (the depth is chosen so that every
                                    rank fits the budget)                                       */
  int64_t acc_rows;              /* rows of this rank's fp32 accumulator (N when world = 1; the
                                    touched blocks of CQS_ACC_BLOCK_ROWS rows when world > 1)   */
  int64_t shard_rows;            /* world > 1: rows of this rank's output shard (cqs_shard_rows) */
} cqs_plan_info_t;

typedef struct {
  int32_t nseg;                        /* maximal segments of consecutive tokens, constant codes */
  int32_t rank;                        /* owning rank (-1 if empty)                              */
  int32_t depth;                       /* leaf depth (quorum[0..depth) is its path from the root) */
  int32_t reserved;
  uint64_t work;                       /* kept (query, key) pairs                                */
  int32_t quorum[CQS_MAX_DEPTH];       /* (q_1..q_depth)                                   */
  int64_t seg_start[CQS_MAX_SEGS];     /* global token id of the segment's first token          */
  int64_t seg_len[CQS_MAX_SEGS];
  uint8_t seg_codes[CQS_MAX_SEGS][CQS_MAX_DEPTH]; /* code_t = index in I order of its level-t
                                                     chunk; 0 = owner (R4)              */
  uint32_t kept[CQS_MAX_SEGS];         /* kept[a] bit b: query seg a attends key seg b; equals
                                          LocalMaskFromGroupRuns at segment granularity */
} cqs_task_t;

/* Build the plan (host only, synchronous).  Validates I, picks depth, enumerates the c^depth
 * quorum tuples lexicographically (R3), cuts each leaf into segments, derives the kept
 * blocks, work and empty flags, assigns non-empty tasks to ranks by LPT on work, and evaluates the
 * memory model.  Errors: CQS_E_INVALID (bad desc), CQS_E_INFEASIBLE (depth=-1 and nothing fits or
 * explicit depth over budget), CQS_E_UNSUPPORTED (> CQS_MAX_SEGS segments).  *out owned by caller,
 * release with cqs_plan_destroy. */
cqs_status cqs_plan(const cqs_plan_desc* desc, cqs_plan_t** out);
cqs_status cqs_plan_info(const cqs_plan_t* plan, cqs_plan_info_t* info);
/* Task `idx` (0 <= idx < n_tasks, lexicographic order) into *task. */
cqs_status cqs_plan_task(const cqs_plan_t* plan, int64_t idx, cqs_task_t* task);
/* Canonical plan bytes (little endian): "CQSP", u32 version=1, i64 N, i32 c, i32 l, i32 I[l],
 * i32 depth, i64 n_tasks, then per task in lexicographic order: i32 nseg, u64 work,
 * nseg x (i64 start, i64 len, u8 codes[depth]), nseg x u32 kept mask.  A hybrid plan whose
 * leaves differ in depth writes version=2: the same, with i32 leaf depth before each task's nseg
 * and codes[leaf depth] per segment (tasks in DFS order of their quorum paths).  A plan with
 * per-level interest sets writes version=3: "CQSP", u32 3, i64 N, i32 depth, i32 L (= deepest
 * leaf), L x (i32 c_t, i32 l_t, i32 I_t[l_t]), i64 n_tasks, then the version-2 task records.
 * If buf is NULL or *len too small, *len receives the required size and CQS_E_INVALID (buf NULL:
 * CQS_OK) is returned. */
cqs_status cqs_plan_serialize(const cqs_plan_t* plan, void* buf, size_t* len);
void cqs_plan_destroy(cqs_plan_t* plan);

/* Memory model M_dev: predicted device bytes of a forward call with the
 * given depth / accumulator tier / staging buffers.  Pure host arithmetic on the desc. */
cqs_status cqs_memory_model(const cqs_plan_desc* desc, int32_t depth, int32_t acc_depth,
                            int32_t n_stage_buffers, uint64_t* dev_bytes, uint64_t* host_bytes);

/* ---------------------------------------------------------------------------------------------
 * Forward (Algorithm 1 in LSE form: per-task partial (O_i, lse_i) + IndexAdd-merge)
 * --------------------------------------------------------------------------------------------- */
typedef struct {
  double ms_plan, ms_h2d, ms_attn, ms_merge, ms_exchange, ms_total; /* filled when stats != NULL
                                                                       (host wall clock, syncs)  */
  uint64_t bytes_h2d, bytes_d2h, bytes_exchanged;
  uint64_t predicted_peak_bytes;   /* the plan's memory-model prediction (not a measurement: the
                                      library allocates nothing, the caller measures — see
                                      tests/test_gpu_memory.py and bench.py "budget")            */
  int64_t tasks_run, tasks_skipped, kernel_launches;
} cqs_stats;

cqs_status cqs_forward_workspace_size(const cqs_plan_t* plan, size_t* dev_bytes, size_t* host_bytes);

/* Run this rank's tasks.
 *   q, k, v     : [B,H,N,D] of desc.in_dtype at desc.qkv_loc.  qkv_strides = element strides of
 *                 (B, H, N, D); stride D must be 1; device tensors need 16-byte aligned rows
 *                 (TMA).  Streamed (pinned host) tensors must be contiguous.
 *   out         : [B,H,N,D] of desc.out_dtype at desc.out_loc with element strides out_strides
 *                 (stride D = 1).  Written only when world == 1 (else see cqs_partial_view).
 *   lse         : nullable, fp32 [B,H,N] contiguous at desc.out_loc: natural-log sum of
 *                 exp(alpha q.k) over all keys (the FA `softmax_lse`).
 *   scale       : alpha; <= 0 selects 1/sqrt(D).
 *   budget_bytes: the caller's device budget; CQS_E_INFEASIBLE if the plan's predicted peak
 *                 exceeds it (0 = trust the plan).
 *   dev_ws/host_ws: at least cqs_forward_workspace_size() bytes (256-byte aligned); host_ws
 *                 pinned.  With world > 1 dev_ws keeps this rank's fp32 partial accumulator
 *                 after the call.
 * Asynchronous on `stream` unless stats != NULL (then it synchronizes to time stages). */
cqs_status cqs_attention_forward(const cqs_plan_t* plan, const void* q, const void* k,
                                 const void* v, const int64_t qkv_strides[4], void* out,
                                 const int64_t out_strides[4], float* lse, float scale,
                                 uint64_t budget_bytes, void* dev_ws, void* host_ws,
                                 void* stream /* cudaStream_t */, cqs_stats* stats);

/* Pointers to the fp32 partial accumulator inside dev_ws after a world > 1 forward:
 * acc_o [acc_rows][B*H][D], acc_lse [acc_rows][B*H] (natural log; -inf = no contribution yet),
 * acc_rows from cqs_plan_info.  Row layout: see cqs_partial_runs. */
cqs_status cqs_partial_view(const cqs_plan_t* plan, void* dev_ws, float** acc_o, float** acc_lse);

/* Which global rows rank `src_rank`'s accumulator holds (world > 1; every rank builds the same plan,
 * so any rank can ask about any other).  A rank's accumulator keeps the blocks of
 * CQS_ACC_BLOCK_ROWS consecutive rows that contain a query row of one of its tasks (rows of an
 * active query segment), packed in increasing global order: global row g of a held block sits at
 * local row slot(g / CQS_ACC_BLOCK_ROWS) * CQS_ACC_BLOCK_ROWS + g % CQS_ACC_BLOCK_ROWS.  With world
 * = 1 the accumulator is the identity over all N rows.
 *   runs  : receives up to max_runs triplets (global_start, len, local_row) — maximal runs of held
 *           rows inside [row0, row0 + rows), ascending (local rows are consecutive inside a run
 *           and across runs);
 *   n_runs: receives the number of runs (also when runs is NULL / max_runs too small: then
 *           CQS_OK with runs untouched if runs == NULL, CQS_E_INVALID otherwise).
 * Errors: CQS_E_INVALID (bad rank or range). */
cqs_status cqs_partial_runs(const cqs_plan_t* plan, int32_t src_rank, int64_t row0, int64_t rows,
                            int64_t* runs, int64_t max_runs, int64_t* n_runs);

/* The single exchange step of a world > 1 forward (Eq. 3): this plan's rank
 * owns rows [row0, row0 + shard_rows) (cqs_shard_rows) and merges, for each of them, the partial
 * rows of every rank whose accumulator holds it (cqs_partial_runs), then writes the final O / lse.
 *   part_o / part_lse : HOST arrays of `world` device pointers (peer memory from cqs_ipc_open, or
 *                       received all-to-all buffers); rank r's local accumulator row x is read at
 *                       part_o[r] + (x - part_row0[r]) * B*H*D and part_lse[r] + (x - part_row0[r]) *
 *                       B*H (part_row0 HOST array; 0 for a whole mapped accumulator, the first
 *                       local row sent for an all-to-all buffer).
 *   out               : device [B,H,shard_rows,D] of desc.out_dtype, element strides out_strides
 *                       (stride D = 1); row 0 = global row row0.
 *   lse_out           : nullable, device fp32 [B,H,shard_rows] contiguous.
 * One merge kernel per maximal run of rows held by the same set of ranks.  Errors: CQS_E_INVALID
 * (world = 1, NULL pointers), CQS_E_CUDA. */
cqs_status cqs_exchange_merge(const cqs_plan_t* plan, const float* const* part_o,
                              const float* const* part_lse, const int64_t* part_row0, void* out,
                              const int64_t out_strides[4], float* lse_out,
                              void* stream /* cudaStream_t */);

/* ---------------------------------------------------------------------------------------------
 * Backward (Algorithm 2; gradient derivation Appendix D).
 *
 * The paper's backward re-gathers each task's Q/K/V/O/dO/lse, runs an FA backward on
 * the leaf with the GLOBAL lse and Delta = rowsum(dO * O) (so per-leaf probabilities are the global
 * P), and IndexAdds dQ/dK/dV.  Here each task runs two tcgen05 kernels that
 * read the tensors in place through TMA and accumulate into fp32 dQ/dK/dV workspaces:
 *   P = exp(alpha q.k - lse_q),  dP = dO V^T,  dS = P (dP - Delta_q)        on every kept block
 *   dV += P^T dO,  dK += alpha dS^T Q  (one CTA per 128-key tile, loops over the query tiles of the
 *   query segments that keep its key segment);   dQ += alpha dS K  (one CTA per 128-query tile).
 * Resident bf16 plans only (desc.qkv_loc = device, in_dtype = bf16); the plan has the forward's
 * depth and tasks.  Sum over tasks = the dense attention gradient (R19).  With world > 1 each rank
 * runs ITS tasks (LPT, as in the forward) into full-size fp32 partial accumulators that stay in
 * dev_ws (cqs_backward_partial_view); the row owner then sums the ranks' partial rows with
 * cqs_reduce_sum (over peer memory or after an all-to-all) — one exchange, no communication
 * during compute.
 * --------------------------------------------------------------------------------------------- */
/* Device workspace of cqs_attention_backward: Delta/lse [B*H][2][round_up(N,4)] fp32 and three fp32
 * accumulators [N][B*H][D] (dQ, dK, dV), each section 256-byte aligned.  CQS_E_UNSUPPORTED for a
 * plan the backward does not run (see above). */
cqs_status cqs_backward_workspace_size(const cqs_plan_t* plan, size_t* dev_bytes);

/* Gradients of L = sum(dO * O) for the forward O = attention(q, k, v) of this plan.
 *   q, k, v, o, dout : device bf16 [B,H,N,D] with element strides qkv_strides (all five tensors
 *                      share the layout; stride D = 1; 16-byte aligned rows, for TMA).
 *   lse              : device fp32 [B,H,N] contiguous, the forward's natural-log lse.
 *   dq, dk, dv       : device [B,H,N,D] of desc.out_dtype with element strides grad_strides
 *                      (stride D = 1); fully overwritten.  Ignored (may be NULL) when world > 1.
 *   scale            : alpha (<= 0 selects 1/sqrt(D)); must equal the forward's.
 *   dev_ws           : >= cqs_backward_workspace_size() bytes, 256-byte aligned, caller-owned.
 * Asynchronous on `stream` unless stats != NULL (ms_attn = task kernels, ms_merge = prep + cast).
 * Errors: CQS_E_INVALID (NULL / misaligned / bad strides), CQS_E_UNSUPPORTED (plan kind),
 * CQS_E_CUDA (launch failure; cqs_last_error has the CUDA message). */
cqs_status cqs_attention_backward(const cqs_plan_t* plan, const void* q, const void* k,
                                  const void* v, const void* o, const void* dout,
                                  const int64_t qkv_strides[4], const float* lse, void* dq,
                                  void* dk, void* dv, const int64_t grad_strides[4], float scale,
                                  void* dev_ws, void* stream /* cudaStream_t */, cqs_stats* stats);

/* Pointers to the fp32 gradient accumulators inside dev_ws after cqs_attention_backward:
 * dQ, dK, dV, each [N][B*H][D] (token-major, so a row shard is one contiguous block). */
cqs_status cqs_backward_partial_view(const cqs_plan_t* plan, void* dev_ws, float** dq, float** dk,
                                     float** dv);

/* R-way sum (Alg. 2's IndexAdd across ranks), on device: for r < rows, p < B*H,
 *   out[b, h, out_row0 + r, :] = cast_out_dtype( sum_j parts[j][r][p][:] )
 * parts: HOST array of n_parts (1..16) device pointers to [rows][B*H][D] fp32 (16-byte aligned;
 * peer pointers from cqs_ipc_open allowed); out: [B,H,N,D] with element strides out_strides
 * (stride D = 1).  D must be a power of two in [4, 256].  Errors: CQS_E_INVALID. */
cqs_status cqs_reduce_sum(int64_t rows, int32_t B, int32_t H, int32_t D, int32_t n_parts,
                          const float* const* parts, void* out, cqs_dtype out_dtype,
                          const int64_t out_strides[4], int64_t out_row0, void* stream);

/* Rows owned by `rank` for the final merge: [row0, row0 + rows) with row0 = floor(rank N / world). */
cqs_status cqs_shard_rows(int64_t N, int32_t world, int32_t rank, int64_t* row0, int64_t* rows);

/* R-way LSE merge (Eq. 3 with Den_j = exp(lse_j), Num_j = O_j Den_j), on device:
 * for r < rows, p < B*H:   lse = log sum_j exp(lse_j[r,p]);   O = sum_j exp(lse_j - lse) O_j[r,p,:]
 * over j < n_parts (part_o[j]: [rows][B*H][D] fp32, part_lse[j]: [rows][B*H] fp32, device
 * pointers listed in HOST arrays), plus the accumulator (acc_o, acc_lse) when non-NULL, which then
 * receives the result.  -inf parts contribute nothing; all -inf gives O = 0, lse = -inf (R8).
 * If out != NULL the result is also written cast to out_dtype into rows [out_row0, out_row0+rows)
 * of the [B,H,N,D] tensor `out` (element strides out_strides), and lse_out (nullable,
 * [B,H,N] contiguous fp32, row offset out_row0, n_total = N) receives lse.  Errors:
 * CQS_E_INVALID (n_parts < 0, D > 256 or not a multiple of 4, NULL required pointer). */
cqs_status cqs_merge(int64_t rows, int32_t B, int32_t H, int32_t D, int32_t n_parts,
                     const float* const* part_o, const float* const* part_lse, float* acc_o,
                     float* acc_lse, void* out, cqs_dtype out_dtype, const int64_t out_strides[4],
                     int64_t out_row0, int64_t n_total, float* lse_out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Peer-memory plumbing for the multi-GPU exchange (one process per GPU).  The final
 * merge reads every rank's partial accumulator directly over NVLink: each rank exports its
 * workspace with cqs_ipc_handle, peers map it with cqs_ipc_open, and cqs_merge is then launched
 * with peer device pointers as its parts (one kernel = exchange + R-way merge).
 * --------------------------------------------------------------------------------------------- */
/* handle (64 bytes, caller-owned) of the device allocation containing dev_ptr, and dev_ptr's byte
 * offset inside it.  Errors: CQS_E_INVALID (NULL), CQS_E_CUDA (not an exportable allocation). */
cqs_status cqs_ipc_handle(const void* dev_ptr, void* handle, uint64_t* offset);
/* Map a peer's allocation (from cqs_ipc_handle) into this process; *base is its base address. */
cqs_status cqs_ipc_open(const void* handle, void** base);
cqs_status cqs_ipc_close(void* base);

const char* cqs_last_error(void);
int32_t cqs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CQS_H_ */

// Per-task CQS attention kernel, bf16 inputs, sm_100a tcgen05 / TMEM / TMA.
//
// Computes, for every kept (query-segment, key-segment) block of one CQS task, the per-task
// partial of Eq. 2 in the normalised form an FA kernel returns:
//   S = alpha Q K^T (tcgen05.mma, fp32 in TMEM) -> online softmax in registers (exp2, one thread
//   per row) -> P (bf16, written back into TMEM over S) -> O += P V (tcgen05.mma, A from TMEM)
// and merges (O_i, lse_i) straight into the fp32 accumulator (Eq. 3 in LSE form) in the
// epilogue, so partials never round-trip through HBM.
//
// CTA = two 128-row query tiles of one query segment (256 rows) of one (b,h) plane; warp roles:
//   warp 0      TMA producer (Q once, then K/V tiles through a kStages ring)
//   warp 1      MMA issuer (single thread): S_j(t0), S_j(t1), then per j: PV_j(t0), S_{j+1}(t0),
//               PV_j(t1), S_{j+1}(t1) — the two tiles ping-pong so one tile's softmax overlaps
//               the other tile's MMAs
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4-7   softmax + correction + epilogue of tile 0 (thread = row = TMEM lane)
//   warps 8-11  same for tile 1
// Masking is block-level (segment-pair skipping, F3); the only element predicate is the
// tail column bound of a key segment's last tile.  Rows beyond the segment are loaded but never
// stored.  O rescaling is conditional (only when the running max grows by > 8 in log2 units).
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "ptx.cuh"
#include "attn_common.cuh"
#include "task_params.cuh"

namespace cqs {

constexpr int kAttnThreads = 384;

#ifdef CQS_DBG_TIMING   // timing experiment only (tools/timing_probe.py --d64)
__device__ unsigned long long g_cqs_dbg1[16];
#define DBG1_T0(v) const long long v = clock64()
#define DBG1_ADD(i, x) atomicAdd(&g_cqs_dbg1[i], (unsigned long long)(x))
#else
#define DBG1_T0(v)
#define DBG1_ADD(i, x) ((void)0)
#endif
// Rescale guard of the speculative pass: with kSumGuard the pass tracks no row max at all (the
// FMNMX chains cost ~11% of the pass); a row is rescaled (exact max, O and l scaled, pass redone)
// only when its P row sum against the running max exceeds kSumLimit, i.e. some p = 2^(x - m) is
// large.  Any reference max is exact (O / l and lse = m + log2 l are invariant under it); the guard
// only keeps p, l and O far from fp32 overflow (l grows at most by kSumLimit per KV tile).
#ifndef CQS_SUM_GUARD
#define CQS_SUM_GUARD 1
#endif
constexpr bool kSumGuard = CQS_SUM_GUARD != 0;
constexpr float kSumLimit = 65536.0f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units (factor 256)
// setmaxnreg split (see the register note in the kernel): 4 warps at LO, 8 softmax warps at HI
// (56 / 224: no spills; measured +3.9% over 72 / 216 at D = 64: 725 vs 697 TFLOP/s, 3 runs each)
#ifndef CQS_ONE_REG_LO
#define CQS_ONE_REG_LO 56
#define CQS_ONE_REG_HI 224
#endif
static_assert(128 * (168 - CQS_ONE_REG_LO) == 256 * (CQS_ONE_REG_HI - 168), "register split");
// column pairs (i mod 8) whose exp2 runs on the FMA pipe instead of MUFU
// (measured on B200, C2 shape, fused exp loop: MUFU-only is fastest at both head dims — D=64:
// 750 TFLOP/s MUFU-only vs 716 at 1/4 of the pairs emulated, 658 at 1/2, 534 at 3/4; D=128 is
// power-capped and emulation only lowers the clock.  The polynomial stays available for
// experiments via -DCQS_DBG_POLY_MASK.)
#ifdef CQS_DBG_POLY_MASK
template <int D> constexpr uint32_t kPolyMask = CQS_DBG_POLY_MASK;
#else
template <int D> constexpr uint32_t kPolyMask = 0x0;
#endif

// Sequenced exp passes of the two tiles (named barriers 1 / 2, 8 warps each): each tile's pass
// runs alone on its sub-partition's MUFU; the S load (tcgen05.ld) stays outside the sequenced
// region.  (Round 1 sequenced the whole phase including the S load: 651 vs 735 TFLOP/s.)
#ifndef CQS_ONE_SEQ
#define CQS_ONE_SEQ 0
#endif
template <int D>
constexpr bool kPingPong = CQS_ONE_SEQ != 0;

template <int D>
struct AttnCfg {
  static constexpr int kBoxes = D / 64;                // 64-column (128-byte) TMA boxes
  static constexpr int kQBytes = kBM * D * 2;
  static constexpr int kKVBytes = kBN * D * 2;
#ifndef CQS_ONE_STAGES64
#define CQS_ONE_STAGES64 8
#endif
  static constexpr int kStages = D == 128 ? 4 : CQS_ONE_STAGES64;
  static constexpr int kSmemBytes = 2 * kQBytes + kStages * kKVBytes + 1024 + 512;
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 256 + D;
  // D = 64: Q lives in TMEM (A operand of S = Q K^T from TMEM, kind::f16 packed like P), so the
  // S MMA reads only K from shared memory (an SS MMA at M = N = 128 needs the full 128 B/clk of
  // SMEM bandwidth, leaving none for the TMA fills).  D = 128 has no free TMEM columns for it.
  static constexpr bool kQInTmem = D == 64;
  static constexpr uint32_t kColQ0 = 256 + 2 * D, kColQ1 = 256 + 2 * D + D / 2;
};

template <int D>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_bf16_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV,
                           const __grid_constant__ TaskParams tp, float* __restrict__ acc_o,
                           float* __restrict__ acc_lse, float scale_log2) {
  using C = AttnCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // [2][kBoxes][128 rows][128 B]
  uint8_t* sKV = smem + 2 * C::kQBytes;       // [kStages][kBoxes][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kStages * C::kKVBytes);
  uint64_t* q_full = bars;                    // 1
  uint64_t* kv_full = bars + 1;               // kStages
  uint64_t* kv_empty = kv_full + C::kStages;  // kStages
  uint64_t* s_full = kv_empty + C::kStages;   // 2
  uint64_t* p_full = s_full + 2;              // 2
  uint64_t* o_bar = p_full + 2;               // 2
  uint64_t* q_tm = o_bar + 2;                 // 1: Q copied into TMEM (kQInTmem)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_tm + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work item: (query segment, 256-row pair) x (b,h) plane ----
  // head-major rasterization: the ~148 CTAs in flight work on the same (b,h) plane and stream the
  // same K/V tiles, so K/V come from L2 instead of being re-read from HBM by every CTA
  const int bh = blockIdx.x / tp.n_items, item = blockIdx.x % tp.n_items;
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  const int a = tp.order[oi];
  const int q_off = (item - (oi ? tp.item_end[oi - 1] : 0)) * (2 * kBM);
  const int len_a = tp.seg_len[a];
  const int valid0 = min(kBM, len_a - q_off);
  const int valid1 = max(0, min(kBM, len_a - q_off - kBM));
  const bool two = valid1 > 0;
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t kmask = tp.kept[a];
  int n_kv = 0;
  for (uint32_t m = kmask; m; m &= m - 1) n_kv += (tp.seg_len[__ffs(m) - 1] + kBN - 1) / kBN;
  const int kv0 = kv_start(item, n_kv);

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 4);
      ptx::mbar_init(&o_bar[t], 1);
    }
    ptx::mbar_init(q_tm, two ? 8 : 4);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // register split (launch: 384 x 168): the 4 non-math warps give back 128 x (168-LO) registers,
  // exactly what the 8 softmax warps take (256 x (HI-168)); .inc blocks forever if the pool is
  // short, so the two numbers must balance (static_assert above).
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CQS_ONE_REG_LO) : "memory");
  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmQ);
      ptx::tma_prefetch_desc(&tmK);
      ptx::tma_prefetch_desc(&tmV);
      const int q_row = tp.seg_src[a] + q_off;
      ptx::mbar_arrive_expect_tx(q_full, (two ? 2 : 1) * C::kQBytes);
      for (int t = 0; t < (two ? 2 : 1); ++t)
        for (int bx = 0; bx < C::kBoxes; ++bx)
          ptx::tma_load_4d(sQ + t * C::kQBytes + bx * kBM * 128, &tmQ, q_full, bx * 64,
                           q_row + t * kBM, hi, bi);
      int it = 0;
      auto load = [&](const CUtensorMap* map, int row) {
        const int s = it % C::kStages;
        const uint32_t ph = (it / C::kStages) & 1;
        ptx::mbar_wait(&kv_empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[s], C::kKVBytes);
        for (int bx = 0; bx < C::kBoxes; ++bx)
          ptx::tma_load_4d(sKV + s * C::kKVBytes + bx * kBN * 128, map, &kv_full[s], bx * 64, row,
                           hi, bi);
        ++it;
      };
      KvCursor ck, cv;
      ck.init(&tp, kmask, kv0);
      cv.init(&tp, kmask, kv0);
      load(&tmK, ck.row());
      ck.next();
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          load(&tmK, ck.row());
          ck.next();
        }
        load(&tmV, cv.row());
        cv.next();
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (whole warp, one elected lane issues) =================
    {
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(kBM, kBN, 0, 0);
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(kBM, D, 0, 1);
      const uint64_t dq0 = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 16, 1024);
      const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), 16, 1024);
      const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), kBN * 128, 1024);
      auto issue_S = [&](int t, int s) {
        const uint64_t qa = dq0 + uint64_t((t * C::kQBytes) >> 4);
        const uint64_t kb = dkv0 + uint64_t((s * C::kKVBytes) >> 4);
        const uint32_t d = tmem + (t ? C::kColS1 : C::kColS0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = ((ks >> 2) * (kBM * 128) + (ks & 3) * 32) >> 4;
          if constexpr (C::kQInTmem)
            ptx::mma_ts_elect(d, tmem + (t ? C::kColQ1 : C::kColQ0) + ks * 8, kb + off, idesc_qk,
                              ks > 0);
          else
            ptx::mma_ss_elect(d, qa + off, kb + off, idesc_qk, ks > 0);
        }
        ptx::mma_commit_elect(&s_full[t]);
      };
      auto issue_PV = [&](int t, int s, bool acc) {
        const uint64_t vb = dv0 + uint64_t((s * C::kKVBytes) >> 4);
        const uint32_t d = tmem + (t ? C::kColO1 : C::kColO0), pa = tmem + (t ? C::kColS1 : C::kColS0);
#pragma unroll
        for (int ks = 0; ks < kBN / 16; ++ks)
          ptx::mma_ts_elect(d, pa + ks * 8, vb + uint64_t((ks * 16 * 128) >> 4), idesc_pv,
                            (acc || ks > 0));
        ptx::mma_commit_elect(&o_bar[t]);
      };
      DBG1_T0(tm0);
      long long mma_pwait = 0, mma_kvwait = 0;
      (void)mma_pwait;
      (void)mma_kvwait;
      int it = 0;
      ptx::mbar_wait(C::kQInTmem ? q_tm : q_full, 0);
      const int sK0 = it % C::kStages;
      ptx::mbar_wait(&kv_full[sK0], (it / C::kStages) & 1);
      ++it;
      ptx::tc_fence_after();
      issue_S(0, sK0);
      if (two) issue_S(1, sK0);
      ptx::mma_commit_elect(&kv_empty[sK0]);
      for (int j = 0; j < n_kv; ++j) {
        int sKn = -1;
        if (j + 1 < n_kv) {
          sKn = it % C::kStages;
          ptx::mbar_wait(&kv_full[sKn], (it / C::kStages) & 1);
          ++it;
        }
        const int sV = it % C::kStages;
        DBG1_T0(tk0);
        ptx::mbar_wait(&kv_full[sV], (it / C::kStages) & 1);
        DBG1_T0(tk1);
#ifdef CQS_DBG_TIMING
        mma_kvwait += tk1 - tk0;
#endif
        ++it;
        ptx::tc_fence_after();
        for (int t = 0; t < (two ? 2 : 1); ++t) {
          DBG1_T0(tw0);
          ptx::mbar_wait(&p_full[t], j & 1);
          DBG1_T0(tw1);
#ifdef CQS_DBG_TIMING
          mma_pwait += tw1 - tw0;
#endif
          ptx::tc_fence_after();
          issue_PV(t, sV, j > 0);
          if (sKn >= 0) issue_S(t, sKn);
        }
        ptx::mma_commit_elect(&kv_empty[sV]);
        if (sKn >= 0) ptx::mma_commit_elect(&kv_empty[sKn]);
      }
      DBG1_T0(tm1);
      if (lane == 0) DBG1_ADD(5, tm1 - tm0), DBG1_ADD(6, n_kv), DBG1_ADD(4, mma_pwait),
                     DBG1_ADD(3, mma_kvwait);
      // drain: q_full's second phase completes when every MMA of this CTA has retired
      ptx::mma_commit_elect(q_full);
      ptx::mbar_wait(q_full, 1);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CQS_ONE_REG_HI) : "memory");
    // ================= softmax / correction / epilogue =================
    const int t = (warp - 4) >> 2;
    if (t == 0 || two) {
      const int sub = warp & 3;
      const int r = sub * 32 + lane;
      const uint32_t lane_base = uint32_t(sub * 32) << 16;
      const uint32_t tS = tmem + lane_base + (t ? C::kColS1 : C::kColS0);
      const uint32_t tO = tmem + lane_base + (t ? C::kColO1 : C::kColO0);
      float m = -INFINITY, l = 0.f;
      const uint32_t a_sfull = ptx::smem_u32(&s_full[t]), a_pfull = ptx::smem_u32(&p_full[t]);
      if constexpr (C::kQInTmem) {
        // this thread's Q row (SW128 TMA box: 16-byte chunk c of row r sits at chunk c ^ (r & 7))
        // -> 32 packed bf16 pairs -> TMEM columns kColQ_t (same packing as P)
        ptx::mbar_wait(q_full, 0);
        const uint8_t* qrow = sQ + t * C::kQBytes + r * 128;
        uint32_t qv[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 u = *reinterpret_cast<const uint4*>(qrow + ((c ^ (r & 7)) << 4));
          qv[4 * c + 0] = u.x, qv[4 * c + 1] = u.y, qv[4 * c + 2] = u.z, qv[4 * c + 3] = u.w;
        }
        ptx::tmem_st32(tmem + lane_base + (t ? C::kColQ1 : C::kColQ0), qv);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(q_tm);
      }
      KvCursor cur;
      cur.init(&tp, kmask, kv0);
      for (int j = 0; j < n_kv; ++j) {
        const int valid = cur.valid();
        cur.next();
        DBG1_T0(ts0);
        ptx::mbar_wait_a(a_sfull, j & 1);
        ptx::tc_fence_after();
        DBG1_T0(ts1);
        uint32_t sr[kBN];
#pragma unroll
        for (int c = 0; c < kBN / 32; ++c)
          ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        ptx::tmem_ld_wait();
        float* s = reinterpret_cast<float*>(sr);
        if (valid < kBN) {
#pragma unroll
          for (int c = 0; c < kBN; ++c)
            if (c >= valid) s[c] = -INFINITY;
        }
        if (kPingPong<D> && two && !(t == 0 && j == 0)) ptx::named_bar_sync(1 + t, 256);
        // One exp2 pass: p = 2^(s*scale_log2 - m_use) (packed FFMA2 argument, MUFU.EX2 — or the
        // FMA-pipe polynomial for the pairs in kPolyMask), fused per 32-column chunk with the
        // packed row sum, the bf16 pack and the tcgen05.st of P.  With TRACK it also takes the
        // row max of the raw scores on the side (speculative max, see below).
        auto exp_pass = [&](float m_use, auto track, float& rmax) -> float {
          constexpr bool kTrack = decltype(track)::value;
          const uint64_t sc2 = ptx::f2(scale_log2, scale_log2), nm2 = ptx::f2(-m_use, -m_use);
          uint64_t rs2[4] = {0, 0, 0, 0};
          float mx4[4];
          if (kTrack) {
#pragma unroll
            for (int u = 0; u < 4; ++u) mx4[u] = -INFINITY;
          }
#pragma unroll
          for (int c = 0; c < kBN / 32; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int ii = 0; ii < 16; ++ii) {
              const int i = 16 * c + ii;
              if (kTrack && (ii & 1) == 0)
                mx4[(i >> 1) & 3] = fmaxf(mx4[(i >> 1) & 3],
                                          fmaxf(fmaxf(s[2 * i], s[2 * i + 1]),
                                                fmaxf(s[2 * i + 2], s[2 * i + 3])));
              float x0, x1;
              ptx::f2_split(ptx::ffma2(ptx::f2(s[2 * i], s[2 * i + 1]), sc2, nm2), x0, x1);
              if ((kPolyMask<D> >> (i & 7)) & 1) {
                ptx::exp2_poly_pair(x0, x1);
                if (2 * i >= valid) x0 = 0.f;         // masked tail columns (poly gives 2^-125)
                if (2 * i + 1 >= valid) x1 = 0.f;
              } else {
                x0 = ptx::ex2(x0);
                x1 = ptx::ex2(x1);
              }
              rs2[ii & 3] = ptx::fadd2(rs2[ii & 3], ptx::f2(x0, x1));
              pk[ii] = ptx::pack_bf16(x0, x1);
            }
            ptx::tmem_st16(tS + c * 16, pk);
          }
          if (kTrack) rmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
          const uint64_t rr = ptx::fadd2(ptx::fadd2(rs2[0], rs2[1]), ptx::fadd2(rs2[2], rs2[3]));
          float a0, a1;
          ptx::f2_split(rr, a0, a1);
          return a0 + a1;
        };
        float rowsum = 0.f, rmax = 0.f;
        bool exact_pass = true;
        auto row_max = [&]() {   // exact raw row max of the tile (8 FMNMX3 chains, then a tree)
          float mx8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) mx8[u] = s[u];
#pragma unroll
          for (int c = 8; c + 16 <= kBN; c += 16) {
#pragma unroll
            for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], fmaxf(s[c + u], s[c + 8 + u]));
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], s[kBN - 8 + u]);   // last 8 columns
          return fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        };
        if (j == 0) {
          m = row_max() * scale_log2;   // first tile: exact row max first
        } else {
          // speculative max: exponentiate against the running max right away and take this
          // tile's max on the side; only when it exceeds m by more than the threshold (rare after
          // the first tiles) are O and l rescaled (O must hold PV_{j-1}) and the pass redone
          rowsum = exp_pass(m, std::bool_constant<!kSumGuard>{}, rmax);
          bool need;
          float mx = 0.f;
          if (kSumGuard) {
            need = !(rowsum <= kSumLimit);   // some p > kSumLimit / kBN (also inf)
          } else {
            mx = rmax * scale_log2;
            need = mx > m + kRescaleThreshold;
          }
          exact_pass = __any_sync(0xffffffffu, need);
          if (exact_pass) {
            if (kSumGuard) {   // rare path: one FMNMX chain (few live registers)
              mx = s[0];
#pragma unroll
              for (int c = 1; c < kBN; ++c) mx = fmaxf(mx, s[c]);
              mx *= scale_log2;
            }
            const float m_new = need ? fmaxf(m, mx) : m;
            ptx::tmem_st_wait();
            ptx::mbar_wait(&o_bar[t], (j - 1) & 1);   // O must hold PV_{j-1}
            ptx::tc_fence_after();
            const float f = need ? ptx::ex2(m - m_new) : 1.f;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t ov[32];
              ptx::tmem_ld32(tO + c * 32, ov);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * f);
              ptx::tmem_st32(tO + c * 32, ov);
            }
            ptx::tmem_st_wait();
            l *= f;
            m = m_new;
          }
        }
        if (exact_pass) rowsum = exp_pass(m, std::false_type{}, rmax);
        if (kPingPong<D> && two && j == 0 && !(t == 1 && j == n_kv - 1))
          ptx::named_bar_arrive(2 - t, 256);
        l += rowsum;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_a(a_pfull);
#ifdef CQS_DBG_TIMING
        DBG1_T0(ts2);
        if (lane == 0) DBG1_ADD(0, ts1 - ts0), DBG1_ADD(1, ts2 - ts1), DBG1_ADD(2, 1);
#endif
      }
      // ---- epilogue: O_i = O / l, lse_i = ln(sum exp) -> merge into the accumulator ----
      ptx::mbar_wait(&o_bar[t], (n_kv - 1) & 1);
      ptx::tc_fence_after();
      const int vrows = t ? valid1 : valid0;
      const bool live = r < vrows;
      const float inv_l = 1.f / l;
      const float lse = (m + __log2f(l)) * 0.69314718055994531f;
      const int64_t idx = int64_t(tp.seg_dst[a] + q_off + t * kBM + r) * tp.BH + bh;
      MergeW w{};
      if (live) w = merge_weights(acc_lse[idx], lse);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(tO + c * 32, ov);
        ptx::tmem_ld_wait();
        if (live) {
          float o[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(ov[i]) * inv_l;
          merge_chunk<32>(acc_o + idx * D + c * 32, o, w);
        }
      }
      if (live) acc_lse[idx] = w.lse;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int D>
static cudaError_t launch_bf16_impl(const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                                    float* acc_lse, float scale, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  auto kern = attn_bf16_sm100_kernel<D>;
  cudaError_t e = set_smem_attr_once(kern, AttnCfg<D>::kSmemBytes, configured);
  if (e != cudaSuccess) return e;
  const int64_t grid = int64_t(tp.n_items) * tp.BH;
  if (grid <= 0) return cudaSuccess;
  kern<<<dim3(unsigned(grid)), kAttnThreads, AttnCfg<D>::kSmemBytes, stream>>>(
      maps[0], maps[1], maps[2], tp, acc_o, acc_lse, scale * 1.4426950408889634f);
  return cudaGetLastError();
}

cudaError_t launch_attn_bf16_pair(const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                                  float* acc_lse, float scale, cudaStream_t stream);
cudaError_t launch_attn_bf16_3t(const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                                float* acc_lse, float scale, cudaStream_t stream);

// D = 128 runs on CTA pairs (cta_group::2, 512 query rows per item; K maps with 64-row boxes);
// D = 64 on the two-tile kernel above (a double-buffered-S alternative measured 680 vs 695
// TFLOP/s on C2-d64; kept out of the build in tools/experiments/attn_bf16_sm100_d64.cu).
// Callers size work items with attn_rows_per_item and build the Q / K / V maps with
// attn_box_rows(D, 0 / 1 / 2).
// D = 64 runs on the three-tile kernel (attn_bf16_sm100_3t.cu: 384 query rows per CTA, 96-key
// K/V tiles) unless built with -DCQS_D64_3T=0 (the two-tile kernel above, 256 rows, 128 keys).
#ifndef CQS_D64_3T
#define CQS_D64_3T 1
#endif
#ifndef CQS_T3_TILES
#define CQS_T3_TILES 3
#define CQS_T3_BN 96
#endif
int attn_rows_per_item(int D) {
  if (D == 128) return 512;
  return CQS_D64_3T ? 128 * CQS_T3_TILES : 256;
}
int attn_box_rows(int D, int which) {
  if (D == 128 && which == 1) return 64;
  if (D == 64 && CQS_D64_3T && which != 0) return CQS_T3_BN;
  return 128;
}

cudaError_t launch_attn_bf16(int D, const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                             float* acc_lse, float scale, cudaStream_t stream) {
  if (D == 128) return launch_attn_bf16_pair(maps, tp, acc_o, acc_lse, scale, stream);
  if (D == 64 && CQS_D64_3T) return launch_attn_bf16_3t(maps, tp, acc_o, acc_lse, scale, stream);
  if (D == 64) return launch_bf16_impl<64>(maps, tp, acc_o, acc_lse, scale, stream);
  return cudaErrorInvalidValue;
}

}  // namespace cqs

#ifdef CQS_DBG_TIMING
extern "C" int cqs_dbg1_read(unsigned long long* out, int n) {
  return int(cudaMemcpyFromSymbol(out, cqs::g_cqs_dbg1, sizeof(unsigned long long) * (n < 16 ? n : 16)));
}
extern "C" int cqs_dbg1_reset() {
  unsigned long long z[16] = {};
  return int(cudaMemcpyToSymbol(cqs::g_cqs_dbg1, z, sizeof(z)));
}
#endif

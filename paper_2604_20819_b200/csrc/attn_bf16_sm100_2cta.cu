// Per-task CQS attention kernel for D = 128 on a CTA PAIR (tcgen05 cta_group::2, M = 256).
//
// Same math and contract as attn_bf16_sm100.cu (Eq. 2 partial in FA form, P:43 / P:240, merged
// into the fp32 accumulator in the epilogue, Eq. 3), but each MMA spans two SMs:
//   S_t = Q_t K^T : M = 256 query rows (128 per CTA, A from each CTA's smem), N = 128 keys split
//                   64 / 64 between the CTAs' smem (B operand), fp32 result: each CTA's TMEM
//                   holds its 128 rows x 128 keys
//   O_t += P_t V  : A = P from each CTA's TMEM, B = V split by head-dim columns 64 / 64
// so every SM stages only HALF of each K and V tile (TMA and shared-memory operand traffic per SM
// halve vs the 1-CTA kernel: measured 1-CTA pure-MMA ceiling was 76% of the tensor peak).
//
// Cluster (2,1,1) = one work item = 512 query rows of one query segment of one (b,h) plane:
// CTA r, tile t owns rows base + 256 t + 128 r.  Warp roles per CTA as in the 1-CTA kernel
// (TMA producer, MMA issuer [leader CTA only], TMEM allocator, 2 x 4 softmax warps).  Barrier
// protocol: kv_full / q_full / p_full live in the LEADER (both CTAs' TMA bytes and both CTAs'
// softmax arrivals land there); s_full / o_bar / kv_empty exist in both CTAs and are signalled by
// the leader's multicast tcgen05.commit.
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "attn_common.cuh"
#include "ptx.cuh"

namespace cqs {

namespace pair {
constexpr int D = 128;
constexpr int kThreads = 384;
constexpr int kQBytes = kBM * D * 2;           // one 128-row Q tile (two 64-col boxes)
constexpr int kKHalfRows = kBN / 2;            // keys per CTA in a K tile
constexpr int kStageBytes = 16384;             // K half (2 boxes of 64 rows) or V half (1 box)
#ifndef CQS_PAIR_STAGES
#define CQS_PAIR_STAGES 8
#endif
constexpr int kStages = CQS_PAIR_STAGES;
constexpr int kSmemBytes = 2 * kQBytes + kStages * kStageBytes + 1024 + 512;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 384;
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
constexpr float kRescaleThreshold = 8.0f;
// setmaxnreg split of the 384 x 168 launch registers: 4 producer / MMA / allocator warps at LO,
// 8 softmax warps at HI, with 128 (168 - LO) = 256 (HI - 168) (an unbalanced .inc blocks forever)
// (56 / 224: no spills; measured +1.7% over 72 / 216 on C2: 1129 vs 1110 TFLOP/s, 3 runs each)
#ifndef CQS_PAIR_REG_LO
#define CQS_PAIR_REG_LO 56
#define CQS_PAIR_REG_HI 224
#endif
static_assert(128 * (168 - CQS_PAIR_REG_LO) == 256 * (CQS_PAIR_REG_HI - 168), "register split");
// Any-order MMA service: the MMA warp serves the two tiles in the order their P becomes ready
// (try_wait polling) instead of strictly tile 0 then tile 1.
#ifndef CQS_PAIR_ANYORDER
#define CQS_PAIR_ANYORDER 0
#endif
constexpr bool kAnyOrder = CQS_PAIR_ANYORDER != 0;
// (Measured and dropped in round 2, all neutral or slower on C2 — profiles/r02_notes.md:
// alternating the two tiles' exp passes with named barriers, storing P after the whole pass,
// releasing P to the MMA in two parts with a deferred rescale.)
// column pairs (i mod 8) whose exp2 runs as an FMA-pipe polynomial instead of MUFU.EX2
#ifdef CQS_DBG_POLY_MASK
constexpr uint32_t kPolyMask = CQS_DBG_POLY_MASK;
#else
constexpr uint32_t kPolyMask = 0x0;
#endif
}  // namespace pair

#ifdef CQS_DBG_TIMING   // timing experiment only: per-role cycle accounting (tools/timing_probe.py)
__device__ unsigned long long g_cqs_dbg[32];
#define DBG_T0(v) const long long v = clock64()
#define DBG_ADD(i, x) atomicAdd(&g_cqs_dbg[i], (unsigned long long)(x))
#else
#define DBG_T0(v)
#define DBG_ADD(i, x)
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair::kThreads, 1)
    attn_bf16_sm100_2cta_kernel(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK,   // box 64 x 64
                                const __grid_constant__ CUtensorMap tmV,   // box 64 x 128
                                const __grid_constant__ TaskParams tp, float* __restrict__ acc_o,
                                float* __restrict__ acc_lse, float scale_log2) {
  using namespace pair;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                                  // [2 tiles][2 boxes][128][128 B]
  uint8_t* sKV = smem + 2 * kQBytes;                   // [kStages][16 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kStageBytes);
  uint64_t* q_full = bars;                             // leader: Q bytes of both CTAs; + drain
  uint64_t* kv_full = bars + 1;                        // leader: K/V half bytes of both CTAs
  uint64_t* kv_empty = kv_full + kStages;              // both: stage free (multicast commit)
  uint64_t* s_full = kv_empty + kStages;               // both: S_t ready (multicast commit)
  uint64_t* p_full = s_full + 2;                       // leader: 8 softmax warps of the pair
  uint64_t* o_bar = p_full + 2;                        // both: PV_t retired (multicast commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef CQS_DBG_TIMING
  const long long k_c0 = clock64();
  unsigned long long k_g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(k_g0));
#endif
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;

  // ---- work item: cluster id -> (b,h) plane (head-major) x (query segment, 512-row block) ----
  const int cid = blockIdx.x >> 1;
  const int bh = cid / tp.n_items, item = cid % tp.n_items;
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  const int a = tp.order[oi];
  const int q_off = (item - (oi ? tp.item_end[oi - 1] : 0)) * (4 * kBM);
  const int len_a = tp.seg_len[a];
  const bool two = len_a - q_off > 2 * kBM;            // tile 1 has rows in either CTA
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t kmask = tp.kept[a];
  int n_kv = 0;
  for (uint32_t m = kmask; m; m &= m - 1) n_kv += (tp.seg_len[__ffs(m) - 1] + kBN - 1) / kBN;
  const int kv0 = kv_start(item, n_kv);

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 8);
      ptx::mbar_init(&o_bar[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();      // barriers of both CTAs initialised, TMEM allocated in both
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CQS_PAIR_REG_LO) : "memory");
    if (warp == 0 && lane == 0) {
      // ================= TMA producer (both CTAs) =================
      ptx::tma_prefetch_desc(&tmQ);
      ptx::tma_prefetch_desc(&tmK);
      ptx::tma_prefetch_desc(&tmV);
      const int q_row = tp.seg_src[a] + q_off + int(rank) * kBM;
      const int ntile = two ? 2 : 1;
      if (leader) ptx::mbar_arrive_expect_tx(q_full, 2 * ntile * kQBytes);
      for (int t = 0; t < ntile; ++t)
        for (int bx = 0; bx < 2; ++bx)
          ptx::tma_load_4d_2sm(sQ + t * kQBytes + bx * kBM * 128, &tmQ, q_full, bx * 64,
                               q_row + t * 2 * kBM, hi, bi);
      int it = 0;
      auto stage_wait = [&](int s) {
        ptx::mbar_wait(&kv_empty[s], ((it / kStages) & 1) ^ 1);
        if (leader) ptx::mbar_arrive_expect_tx(&kv_full[s], 2 * kStageBytes);
        return true;
      };
      KvCursor ck, cv;
      ck.init(&tp, kmask, kv0);
      cv.init(&tp, kmask, kv0);
      auto load_k = [&]() {   // keys [64 rank, 64 rank + 64) of the tile, both 64-col boxes
        const int s = it % kStages;
        if (stage_wait(s))
        for (int bx = 0; bx < 2; ++bx)
          ptx::tma_load_4d_2sm(sKV + s * kStageBytes + bx * kKHalfRows * 128, &tmK, &kv_full[s],
                               bx * 64, ck.row() + int(rank) * kKHalfRows, hi, bi);
        ck.next();
        ++it;
      };
      auto load_v = [&]() {   // head-dim columns [64 rank, 64 rank + 64) of all 128 keys
        const int s = it % kStages;
        if (stage_wait(s))
        ptx::tma_load_4d_2sm(sKV + s * kStageBytes, &tmV, &kv_full[s], int(rank) * 64, cv.row(),
                             hi, bi);
        cv.next();
        ++it;
      };
      load_k();
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) load_k();
        load_v();
      }
    } else if (warp == 1 && leader) {
      // ================= MMA issuer (leader CTA; whole warp, one elected lane issues) =================
      // Descriptors are precomputed: the smem start address lives in the low 14 bits (addr >> 4),
      // so a byte offset is added as offset >> 4 (all offsets stay inside the 227 KB window).
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(2 * kBM, kBN, 0, 0);   // M=256, N=128
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(2 * kBM, D, 0, 1);     // M=256, N=128
      const uint64_t dq0 = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 16, 1024);
      const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), 16, 1024);
      const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), kBN * 128, 1024);
      auto issue_S = [&](int t, int s) {
        const uint64_t qa = dq0 + uint64_t((t * kQBytes) >> 4);
        const uint64_t kb = dkv0 + uint64_t((s * kStageBytes) >> 4);
        const uint32_t d = tmem + (t ? kColS1 : kColS0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t qo = ((ks >> 2) * (kBM * 128) + (ks & 3) * 32) >> 4;
          const uint32_t ko = ((ks >> 2) * (kKHalfRows * 128) + (ks & 3) * 32) >> 4;
          ptx::mma_ss_2sm_elect(d, qa + qo, kb + ko, idesc_qk, ks > 0);
        }
        ptx::mma_commit_2sm_elect(&s_full[t]);
      };
      auto issue_PV = [&](int t, int s, bool acc) {
        const uint64_t vb = dv0 + uint64_t((s * kStageBytes) >> 4);
        const uint32_t d = tmem + (t ? kColO1 : kColO0), pa = tmem + (t ? kColS1 : kColS0);
#pragma unroll
        for (int ks = 0; ks < kBN / 16; ++ks)
          ptx::mma_ts_2sm_elect(d, pa + ks * 8, vb + uint64_t((ks * 16 * 128) >> 4), idesc_pv,
                                (acc || ks > 0));
        ptx::mma_commit_2sm_elect(&o_bar[t]);
      };
      int it = 0;
#ifdef CQS_DBG_TIMING
      long long mma_pwait = 0;
#endif
      DBG_T0(tm0);
      ptx::mbar_wait(q_full, 0);
      const int sK0 = it % kStages;
      ptx::mbar_wait(&kv_full[sK0], (it / kStages) & 1);
      ++it;
      ptx::tc_fence_after();
      issue_S(0, sK0);
      if (two) issue_S(1, sK0);
      ptx::mma_commit_2sm_elect(&kv_empty[sK0]);
      for (int j = 0; j < n_kv; ++j) {
        int sKn = -1;
        if (j + 1 < n_kv) {
          sKn = it % kStages;
          ptx::mbar_wait(&kv_full[sKn], (it / kStages) & 1);
          ++it;
        }
        const int sV = it % kStages;
        ptx::mbar_wait(&kv_full[sV], (it / kStages) & 1);
        ++it;
        ptx::tc_fence_after();
        auto serve = [&](int t) {   // O_t += P_t V_j, then S_t(j+1) over the consumed P_t
          ptx::tc_fence_after();
          issue_PV(t, sV, j > 0);
          if (sKn >= 0) issue_S(t, sKn);
        };
        int first = 0;   // with kAnyOrder: the tile whose P is ready first is served first
        if (kAnyOrder && two)
          for (;; ) {
            if (ptx::mbar_try_wait(&p_full[0], j & 1)) break;
            if (ptx::mbar_try_wait(&p_full[1], j & 1)) {
              first = 1;
              break;
            }
          }
        for (int k = 0; k < (two ? 2 : 1); ++k) {
          const int t = k ? 1 - first : first;
          DBG_T0(tw0);
          ptx::mbar_wait(&p_full[t], j & 1);
#ifdef CQS_DBG_TIMING
          DBG_T0(tw1);
          mma_pwait += tw1 - tw0;
#endif
          serve(t);
        }
        ptx::mma_commit_2sm_elect(&kv_empty[sV]);
        if (sKn >= 0) ptx::mma_commit_2sm_elect(&kv_empty[sKn]);
      }
      ptx::mma_commit_2sm_elect(q_full);   // drain: all MMAs of the pair retired
      ptx::mbar_wait(q_full, 1);
#ifdef CQS_DBG_TIMING
      DBG_T0(tm1);
      if (lane == 0) DBG_ADD(5, tm1 - tm0), DBG_ADD(6, n_kv), DBG_ADD(4, mma_pwait);
#endif
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CQS_PAIR_REG_HI) : "memory");
    // ================= softmax / correction / epilogue (both CTAs) =================
    const int t = (warp - 4) >> 2;
    if (t == 0 || two) {
      const int sub = warp & 3;
      const int r = sub * 32 + lane;
      const uint32_t lane_base = uint32_t(sub * 32) << 16;
      const uint32_t tS = tmem + lane_base + (t ? kColS1 : kColS0);
      const uint32_t tO = tmem + lane_base + (t ? kColO1 : kColO0);
      float m = -INFINITY, l = 0.f;
      const uint32_t a_sfull = ptx::smem_u32(&s_full[t]), a_pfull = ptx::smem_u32(&p_full[t]);
#ifdef CQS_DBG_TIMING
      long long dc[12] = {};
#endif
      KvCursor cur;
      cur.init(&tp, kmask, kv0);
#ifdef CQS_DBG_TIMING
      const long long tl0 = clock64();
#endif
      for (int j = 0; j < n_kv; ++j) {
        const int valid = cur.valid();
        cur.next();
        DBG_T0(ts0);
        ptx::mbar_wait_a(a_sfull, j & 1);
        ptx::tc_fence_after();
        DBG_T0(ts1);
#ifdef CQS_DBG_TIMING
        dc[0] += ts1 - ts0, dc[2] += 1;
#endif
        uint32_t sr[kBN];
#pragma unroll
        for (int c = 0; c < kBN / 32; ++c)
          ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        ptx::tmem_ld_wait();
        DBG_T0(tp_ld);
        float* s = reinterpret_cast<float*>(sr);
        if (valid < kBN) {
#pragma unroll
          for (int c = 0; c < kBN; ++c)
            if (c >= valid) s[c] = -INFINITY;
        }
        // One exp2 pass: p = 2^(s*scale_log2 - m_use) fused per 32-column chunk with the packed
        // row sum, the bf16 pack and the tcgen05.st of P (sums / packs / stores fill the issue
        // slots between MUFU ops).  With TRACK it also takes the row max of the raw scores on the
        // side (4 FMNMX3 chains on the ALU pipe) — the "speculative max" of step j > 0 below.
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
              if ((kPolyMask >> (i & 7)) & 1) {
                ptx::exp2_poly_pair(x0, x1);
                if (2 * i >= valid) x0 = 0.f;   // masked tail columns (poly gives 2^-125)
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
#ifdef CQS_DBG_TIMING
        long long tp_max = tp_ld, tp_gate = 0, tp_exp = 0;
#define DBG_MARK(v) v = clock64()
#else
#define DBG_MARK(v)
#endif
        bool exact_pass = true;   // run the plain pass against the final m
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
          // speculative max: exponentiate against the running max m right away and take this
          // tile's max on the side; only if it exceeds m by more than the rescale threshold
          // (2^8; rare after the first tiles) are O and l rescaled and the pass redone.
          DBG_MARK(tp_max);
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
        DBG_MARK(tp_gate);
        if (exact_pass) rowsum = exp_pass(m, std::false_type{}, rmax);
        DBG_MARK(tp_exp);
        l += rowsum;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_leader_a(a_pfull);
#ifdef CQS_DBG_TIMING
        {
          const long long tp_end = clock64();
          dc[1] += tp_end - ts1, dc[7] += tp_ld - ts1, dc[8] += tp_max - tp_ld;
          dc[9] += tp_gate - tp_max, dc[10] += tp_exp - tp_gate, dc[11] += tp_end - tp_exp;
        }
#endif
      }
#ifdef CQS_DBG_TIMING
      if (lane == 0)
        for (int i = 0; i < 12; ++i)
          if (i < 3 || i >= 7) DBG_ADD(i, dc[i]);
#endif
      // ---- epilogue ----
      DBG_T0(te0);
#ifdef CQS_DBG_TIMING
      if (lane == 0 && warp == 4) DBG_ADD(16, tl0 - k_c0), DBG_ADD(17, te0 - tl0), DBG_ADD(19, 1);
#endif
      ptx::mbar_wait(&o_bar[t], (n_kv - 1) & 1);
      ptx::tc_fence_after();
      const int row_in_seg = q_off + t * 2 * kBM + int(rank) * kBM + r;
      const bool live = row_in_seg < len_a;
      const float inv_l = 1.f / l;
      const float lse = (m + __log2f(l)) * 0.69314718055994531f;
      const int64_t idx = int64_t(tp.seg_dst[a] + row_in_seg) * tp.BH + bh;
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
#ifdef CQS_DBG_TIMING
      if (lane == 0) DBG_ADD(3, clock64() - te0);
      if (lane == 0 && warp == 4) DBG_ADD(18, clock64() - k_c0);
#endif
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();      // both CTAs done with TMEM / peer barriers before teardown
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tmem, 512);
  }
#ifdef CQS_DBG_TIMING
  if (threadIdx.x == 0) {   // per-CTA lifetime: cycles, ns (-> in-kernel clock, SM occupancy)
    unsigned long long k_g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(k_g1));
    DBG_ADD(12, clock64() - k_c0), DBG_ADD(13, k_g1 - k_g0), DBG_ADD(14, 1);
  }
#endif
}

#ifdef CQS_DBG_TIMING
extern "C" int cqs_dbg_read(unsigned long long* out, int n) {
  return int(cudaMemcpyFromSymbol(out, g_cqs_dbg, sizeof(unsigned long long) * n));
}
extern "C" int cqs_dbg_reset() {
  unsigned long long z[32] = {};
  return int(cudaMemcpyToSymbol(g_cqs_dbg, z, sizeof(z)));
}
#endif

cudaError_t launch_attn_bf16_pair(const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                                  float* acc_lse, float scale, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = set_smem_attr_once(attn_bf16_sm100_2cta_kernel, pair::kSmemBytes, configured);
  if (e != cudaSuccess) return e;
  const int64_t grid = 2 * int64_t(tp.n_items) * tp.BH;
  if (grid <= 0) return cudaSuccess;
  attn_bf16_sm100_2cta_kernel<<<dim3(unsigned(grid)), pair::kThreads, pair::kSmemBytes, stream>>>(
      maps[0], maps[1], maps[2], tp, acc_o, acc_lse, scale * 1.4426950408889634f);
  return cudaGetLastError();
}

}  // namespace cqs

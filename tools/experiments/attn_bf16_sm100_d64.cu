// Per-task CQS attention kernel for D = 64: one 128-row query tile per CTA, DOUBLE-BUFFERED S,
// softmax split by key columns over 8 warps.
//
// STATUS: experiment, built but routed only with -DCQS_D64_DBS.  Parity-green (tests/
// test_gpu_attention.py under that build), measured on C2-d64 (N=131072, H=32, one level):
// 680 TFLOP/s vs 695 for the two-tile kernel, both at the 1 kW power cap (~1.92-1.96 GHz); with
// the K/V multicast cluster (-DCQS_D64_MC) 658 at 958 W.  Cycle counters (tools/timing_probe64.py):
// per 128x128 block 1346 cycles of S->P work + 213 waiting for S against a 1024-cycle MUFU floor.
//
// Same math and contract as attn_bf16_sm100.cu (the per-task partial of Eq. 2 in FA form, P:43 /
// P:240, merged into the fp32 accumulator in the epilogue, Eq. 3).  Why another
// schedule at D = 64: per 128 x 128 block the tensor work is 512 cycles but the 16384 exp2 take
// 1024 cycles of MUFU, so the kernel is MUFU-bound and the softmax must never wait for S.  In the
// two-tile kernel each tile's softmax waits for its own PV + S round trip (measured: 2349 cycles
// of S->P work + 1491 cycles waiting for S per tile, both tiles in lock step).  Here S_{j+1} is
// computed into the second TMEM buffer while the softmax works on S_j, so the softmax runs back
// to back; the tensor pipe (512 of every 1024 cycles) hides under it.
//
// TMEM (512 columns allocated): S/P buffer 0 [0,128) | S/P buffer 1 [128,256) | O_0 [256,320) |
// O_1 [320,384) | Q [384,416).  Q is copied once from its TMA tile into TMEM so S = Q K^T reads only
// K from SMEM.  P (bf16, packed pairs) of key half h is written over the S columns that half
// read: keys [0,64) -> columns [0,32), keys [64,128) -> columns [64,96) of the buffer.
//
// With -DCQS_D64_MC, clusters of 2 CTAs take 256 consecutive rows of one query segment: each CTA
// loads one 64-row half of every K/V tile and multicasts it to both (half the L2 traffic); a stage
// is refilled once the MMA commits of BOTH CTAs freed it.
//
// Warps: 0 TMA producer | 1 MMA issuer | 2 TMEM allocator | 3 idle |
//        4-7 softmax of keys [0,64) of every tile for rows 32(w&3).. | 8-11 keys [64,128), same rows.
// The two key halves are independent online softmaxes (own running max m_h, sum l_h and TMEM
// accumulator O_h = sum P_h V_h), i.e. the tile's keys are split into two sets whose partials
// are merged in the epilogue exactly like CQS partials (Eq. 3 in LSE form).  Warps w and w+4 share
// a sub-partition and TMEM lanes but never wait for each other inside the loop.
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "attn_common.cuh"
#include "ptx.cuh"
#include "task_params.cuh"

namespace cqs {

namespace d64 {
constexpr int D = 64;
constexpr int kThreads = 384;
constexpr int kQBytes = kBM * D * 2;       // 16 KB, one 128 B-wide SW128 box
constexpr int kKVBytes = kBN * D * 2;      // 16 KB per K or V tile
constexpr int kStages = 10;
constexpr int kSmemBytes = kQBytes + kStages * kKVBytes + 1024 + 512;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 320, kColQ = 384;
constexpr float kRescaleThreshold = 8.0f;  // log2 units (factor 256)
// CQS_D64_MC: 2-CTA clusters sharing K/V tiles by TMA multicast (halves L2->SM traffic and
// power; measured slower on C2-d64: 657 vs 680 TFLOP/s, so off by default)
#ifdef CQS_D64_MC
constexpr int kCl = 2;
#define CQS_D64_CLUSTER __cluster_dims__(2, 1, 1)
#else
constexpr int kCl = 1;
#define CQS_D64_CLUSTER
#endif
// CQS_D64_SKEW: the key-half-1 warps start this many cycles late (phase offset experiment)
#ifndef CQS_D64_SKEW
#define CQS_D64_SKEW 0
#endif
}  // namespace d64

int d64_rows_per_item() { return d64::kCl * kBM; }
int d64_kv_box_rows() { return kBN / d64::kCl; }

#ifdef CQS_DBG_TIMING   // timing experiment only (tools/timing_probe.py --d64)
__device__ unsigned long long g_cqs_dbg64[16];
#define DBG_T0(v) const long long v = clock64()
#define DBG_ADD(i, x) atomicAdd(&g_cqs_dbg64[i], (unsigned long long)(x))
#else
#define DBG_T0(v)
#define DBG_ADD(i, x) ((void)0)
#endif

__global__ void CQS_D64_CLUSTER __launch_bounds__(d64::kThreads, 1)
    attn_bf16_sm100_d64_kernel(const __grid_constant__ CUtensorMap tmQ,
                               const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV,
                               const __grid_constant__ TaskParams tp, float* __restrict__ acc_o,
                               float* __restrict__ acc_lse, float scale_log2) {
  using namespace d64;
  extern __shared__ uint8_t smem_raw[];
  __shared__ float xm[2][kBM], xl[2][kBM];   // [key half][row]: running max / sum (epilogue)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                                  // [128 rows][128 B] SW128
  uint8_t* sKV = smem + kQBytes;                       // [kStages][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kKVBytes);
  uint64_t* q_full = bars;                             // Q TMA bytes; phase 1 = MMA drain
  uint64_t* kv_full = bars + 1;                        // kStages
  uint64_t* kv_empty = kv_full + kStages;              // kStages
  uint64_t* s_full = kv_empty + kStages;               // 2: S in buffer b ready
  uint64_t* p_full = s_full + 2;                       // [b][h]: P of half h in buffer b (4 warps)
  uint64_t* o_bar = p_full + 4;                        // 1: PV_j (both halves) retired
  uint64_t* q_tm = o_bar + 1;                          // 1: Q copied into TMEM (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_tm + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work item (one per cluster): (query segment, 256-row block) x (b,h) plane, head-major;
  // CTA `rank` owns the block's rows [128 rank, 128 rank + 128).  Both CTAs stream the same K/V
  // tiles: each loads one 64-row half of every tile and multicasts it into both CTAs' smem.
  const uint32_t rank = kCl == 2 ? ptx::cluster_ctarank() : 0;
  const int cid = blockIdx.x / kCl;
  const int bh = cid / tp.n_items, item = cid % tp.n_items;
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  const int a = tp.order[oi];
  const int q_off = (item - (oi ? tp.item_end[oi - 1] : 0)) * (kCl * kBM) + int(rank) * kBM;
  const int len_a = tp.seg_len[a];
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t kmask = tp.kept[a];
  int n_kv = 0;
  for (uint32_t m = kmask; m; m &= m - 1) n_kv += (tp.seg_len[__ffs(m) - 1] + kBN - 1) / kBN;
  const int kv0 = kv_start(item, n_kv);

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], kCl);   // freed by the MMA commits of every CTA of the cluster
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[2 * b], 4);
      ptx::mbar_init(&p_full[2 * b + 1], 4);
    }
    ptx::mbar_init(o_bar, 1);
    ptx::mbar_init(q_tm, 4);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  if (kCl == 2)
    ptx::cluster_sync();    // both CTAs' barriers initialised before any multicast lands
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      // ================= TMA producer: Q, then K_0, K_1, (V_j, K_{j+2})... =================
      ptx::tma_prefetch_desc(&tmQ);
      ptx::tma_prefetch_desc(&tmK);
      ptx::tma_prefetch_desc(&tmV);
      ptx::mbar_arrive_expect_tx(q_full, kQBytes);
      ptx::tma_load_4d(sQ, &tmQ, q_full, 0, tp.seg_src[a] + q_off, hi, bi);
      int it = 0;
      auto load = [&](const CUtensorMap* map, int row) {
        const int s = it % kStages;
        ptx::mbar_wait(&kv_empty[s], ((it / kStages) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[s], kKVBytes);   // both halves land here
        if (kCl == 2)
          ptx::tma_load_4d_mc(sKV + s * kKVBytes + int(rank) * (kKVBytes / 2), map, &kv_full[s],
                              0, row + int(rank) * (kBN / 2), hi, bi, 0x3);
        else
          ptx::tma_load_4d(sKV + s * kKVBytes, map, &kv_full[s], 0, row, hi, bi);
        ++it;
      };
      KvCursor ck, cv;
      ck.init(&tp, kmask, kv0);
      cv.init(&tp, kmask, kv0);
      for (int j = 0; j < 2 && j < n_kv; ++j) {
        load(&tmK, ck.row());
        ck.next();
      }
      for (int j = 0; j < n_kv; ++j) {
        load(&tmV, cv.row());
        cv.next();
        if (j + 2 < n_kv) {
          load(&tmK, ck.row());
          ck.next();
        }
      }
    } else if (warp == 1) {
      // ================= MMA issuer (whole warp, one elected lane issues) =================
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(kBM, kBN, 0, 0);   // M=128, N=128
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(kBM, D, 0, 1);     // M=128, N=64
      const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), 16, 1024);
      const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), kBN * 128, 1024);
      int it = 0;
#ifdef CQS_DBG_TIMING
      long long w_kv = 0, w_p = 0;
#endif
      DBG_T0(tm0);
      auto wait_full = [&]() {
        const int s = it % kStages;
        DBG_T0(t0);
        ptx::mbar_wait(&kv_full[s], (it / kStages) & 1);
#ifdef CQS_DBG_TIMING
        w_kv += clock64() - t0;
#endif
        ++it;
        return s;
      };
      auto issue_S = [&](int b, int s) {   // S_b = Q K_s^T, A = Q from TMEM
        const uint64_t kb = dkv0 + uint64_t((s * kKVBytes) >> 4);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          ptx::mma_ts_elect(tmem + (b ? kColS1 : kColS0), tmem + kColQ + ks * 8,
                            kb + uint64_t((ks * 32) >> 4), idesc_qk, ks > 0);
        ptx::mma_commit_elect(&s_full[b]);
        if (kCl == 2) ptx::mma_commit_mc_elect(&kv_empty[s], 0x3);
        else ptx::mma_commit_elect(&kv_empty[s]);
      };
      // O_h += P_{b,h} V_s[keys of half h], A = P from TMEM (half h's packed columns)
      auto issue_PV = [&](int b, int h, int s, bool acc) {
        const uint64_t vb = dv0 + uint64_t((s * kKVBytes) >> 4);
        const uint32_t pa = tmem + (b ? kColS1 : kColS0) + h * 64;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          ptx::mma_ts_elect(tmem + (h ? kColO1 : kColO0), pa + ks * 8,
                            vb + uint64_t(((4 * h + ks) * 16 * 128) >> 4), idesc_pv, acc || ks > 0);
      };
      ptx::mbar_wait(q_tm, 0);
      for (int j = 0; j < 2 && j < n_kv; ++j) {
        const int s = wait_full();
        ptx::tc_fence_after();
        issue_S(j, s);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const int sV = wait_full();
        for (int h = 0; h < 2; ++h) {
          DBG_T0(tp0);
          ptx::mbar_wait(&p_full[2 * b + h], (j >> 1) & 1);
#ifdef CQS_DBG_TIMING
          w_p += clock64() - tp0;
#endif
          ptx::tc_fence_after();
          issue_PV(b, h, sV, j > 0);
        }
        ptx::mma_commit_elect(o_bar);
        if (kCl == 2) ptx::mma_commit_mc_elect(&kv_empty[sV], 0x3);
        else ptx::mma_commit_elect(&kv_empty[sV]);
        if (j + 2 < n_kv) {   // S_{j+2} overwrites P_j: issued after PV_j (in-order pipe)
          const int sK = wait_full();
          ptx::tc_fence_after();
          issue_S(b, sK);
        }
      }
      ptx::mma_commit_elect(q_full);   // drain: every MMA of this CTA has retired
      ptx::mbar_wait(q_full, 1);
#ifdef CQS_DBG_TIMING
      if (lane == 0) DBG_ADD(4, w_p), DBG_ADD(5, clock64() - tm0), DBG_ADD(6, n_kv), DBG_ADD(7, w_kv);
#endif
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ================= softmax (key half h of rows r), correction, epilogue =================
    const int h = (warp - 4) >> 2;
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t lane_base = uint32_t(sub * 32) << 16;
    const uint32_t pair_bar = 1 + sub;   // named barrier of warps sub+4 and sub+8
    if (h == 0) {
      // this thread's Q row (SW128: 16-byte chunk c of row r sits at chunk c ^ (r & 7)) ->
      // 32 packed bf16 pairs -> TMEM columns [kColQ, kColQ + 32) (packed like P)
      ptx::mbar_wait(q_full, 0);
      const uint8_t* qrow = sQ + r * 128;
      uint32_t qv[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(qrow + ((c ^ (r & 7)) << 4));
        qv[4 * c + 0] = u.x, qv[4 * c + 1] = u.y, qv[4 * c + 2] = u.z, qv[4 * c + 3] = u.w;
      }
      ptx::tmem_st32(tmem + lane_base + kColQ, qv);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(q_tm);
    }
    // Each key half runs its own online softmax (m_h, l_h, O_h) over its 64 keys of every tile:
    // no per-tile exchange between the two warps of a sub-partition, so their latencies overlap.
    // The two partial results are merged in the epilogue (the LSE merge of Eq. 3).
    // m starts at a finite floor so a half whose keys are all masked so far stays 0-weighted.
    float m = -1e30f, l = 0.f;
    if (CQS_D64_SKEW > 0 && h == 1) {
      const long long t0 = clock64();
      while (clock64() - t0 < CQS_D64_SKEW) {
      }
    }
#ifdef CQS_DBG_TIMING
    long long dc_s = 0, dc_p = 0;
#endif
    const uint32_t tO = tmem + lane_base + (h ? kColO1 : kColO0);
    KvCursor cur;
    cur.init(&tp, kmask, kv0);
    for (int j = 0; j < n_kv; ++j) {
      const int valid = cur.valid() - h * 64;   // valid columns of this half (may be <= 0)
      cur.next();
      const int b = j & 1;
      const uint32_t tS = tmem + lane_base + (b ? kColS1 : kColS0) + h * 64;
      DBG_T0(ts0);
      ptx::mbar_wait(&s_full[b], (j >> 1) & 1);
      ptx::tc_fence_after();
      DBG_T0(ts1);
#ifdef CQS_DBG_TIMING
      dc_s += ts1 - ts0;
#endif
      uint32_t sr[64];
      ptx::tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      ptx::tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      ptx::tmem_ld_wait();
      float* s = reinterpret_cast<float*>(sr);
      if (valid < 64) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c >= valid) s[c] = -INFINITY;
      }
      // p = 2^(s*scale_log2 - m_use) for the 64 columns, fused with the packed row sum, the bf16
      // pack and the tcgen05.st of P; with TRACK also the half-row max of the raw scores.
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
        for (int c = 0; c < 2; ++c) {
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
            x0 = ptx::ex2(x0);
            x1 = ptx::ex2(x1);
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
      float rowsum, rmax = 0.f;
      if (j == 0) {
        // first tile: exact half-row max (8 chains, then a small tree)
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(s[u], s[8 + u]);
#pragma unroll
        for (int c = 16; c < 64; c += 16) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], fmaxf(s[c + u], s[c + 8 + u]));
        }
        const float hm = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        m = fmaxf(hm * scale_log2, -1e30f);
        rowsum = exp_pass(m, std::false_type{}, rmax);
      } else {
        // speculative max: exponentiate against the running max right away; only when the
        // half-row max exceeds m by more than the threshold are O_h and l rescaled (O_h must hold
        // PV_{j-1}) and the pass redone
        rowsum = exp_pass(m, std::true_type{}, rmax);
        const float mx = rmax * scale_log2;
        const bool need = mx > m + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m;
          ptx::tmem_st_wait();
          ptx::mbar_wait(o_bar, (j - 1) & 1);   // phases < j-1 retired before S_j (same pipe)
          ptx::tc_fence_after();
          const float f = need ? ptx::ex2(m - m_new) : 1.f;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(tO + c * 32, ov);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * f);
            ptx::tmem_st32(tO + c * 32, ov);
          }
          l *= f;
          m = m_new;
          rowsum = exp_pass(m, std::false_type{}, rmax);
        }
      }
      l += rowsum;
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[2 * b + h]);
#ifdef CQS_DBG_TIMING
      dc_p += clock64() - ts1;
#endif
    }
#ifdef CQS_DBG_TIMING
    if (lane == 0) DBG_ADD(0, dc_s), DBG_ADD(1, dc_p), DBG_ADD(2, n_kv);
#endif
    // ---- epilogue: merge the two halves (LSE form), O_i = O / l, lse_i -> accumulator ----
    xm[h][r] = m;
    xl[h][r] = l;
    // every MMA retired: the MMA warp's drain commit completes q_full's second phase.  (o_bar
    // cannot be used here: PV_{n_kv-2} may still be in flight, and its parity equals PV_{n_kv}'s.)
    ptx::mbar_wait(q_full, 1);
    ptx::tc_fence_after();
    const int row_in_seg = q_off + r;
    const bool live = row_in_seg < len_a;
    const int64_t idx = int64_t(tp.seg_dst[a] + row_in_seg) * tp.BH + bh;
    ptx::named_bar_sync(pair_bar, 64);   // xm / xl visible; both halves read acc_lse[idx] below
    const float m0 = xm[0][r], m1 = xm[1][r];
    const float mm = fmaxf(m0, m1);
    const float w0 = ptx::ex2(m0 - mm), w1 = ptx::ex2(m1 - mm);
    const float lt = xl[0][r] * w0 + xl[1][r] * w1;
    const float inv_l = 1.f / lt;
    const float lse = (mm + __log2f(lt)) * 0.69314718055994531f;
    MergeW w{};
    if (live) w = merge_weights(acc_lse[idx], lse);
    // this warp finalizes D columns [32h, 32h + 32) from both halves' accumulators
    uint32_t oa[32], ob[32];
    ptx::tmem_ld32(tmem + lane_base + kColO0 + h * 32, oa);
    ptx::tmem_ld32(tmem + lane_base + kColO1 + h * 32, ob);
    ptx::tmem_ld_wait();
    if (live) {
      const float c0 = w0 * inv_l, c1 = w1 * inv_l;
      float o[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        o[i] = __uint_as_float(oa[i]) * c0 + __uint_as_float(ob[i]) * c1;
      merge_chunk<32>(acc_o + idx * D + h * 32, o, w);
    }
    ptx::named_bar_sync(pair_bar, 64);   // both halves have read acc_lse[idx]
    if (live && h == 0) acc_lse[idx] = w.lse;
  }

  ptx::tc_fence_before();
  if (kCl == 2)
    ptx::cluster_sync();    // no multicast / remote arrive may target a CTA that has exited
  else
    __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

cudaError_t launch_attn_bf16_d64(const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                                 float* acc_lse, float scale, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = set_smem_attr_once(attn_bf16_sm100_d64_kernel, d64::kSmemBytes, configured);
  if (e != cudaSuccess) return e;
  const int64_t grid = d64::kCl * int64_t(tp.n_items) * tp.BH;
  if (grid <= 0) return cudaSuccess;
  attn_bf16_sm100_d64_kernel<<<dim3(unsigned(grid)), d64::kThreads, d64::kSmemBytes, stream>>>(
      maps[0], maps[1], maps[2], tp, acc_o, acc_lse, scale * 1.4426950408889634f);
  return cudaGetLastError();
}

}  // namespace cqs

#ifdef CQS_DBG_TIMING
extern "C" int cqs_dbg64_read(unsigned long long* out, int n) {
  return int(cudaMemcpyFromSymbol(out, cqs::g_cqs_dbg64, sizeof(unsigned long long) * (n < 16 ? n : 16)));
}
extern "C" int cqs_dbg64_reset() {
  unsigned long long z[16] = {};
  return int(cudaMemcpyToSymbol(cqs::g_cqs_dbg64, z, sizeof(z)));
}
#endif

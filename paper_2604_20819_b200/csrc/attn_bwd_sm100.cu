// Per-task CQS attention backward kernels, bf16 inputs, sm_100a tcgen05 / TMEM / TMA.
//
// Algorithm 2 runs an FA backward on every leaf with the GLOBAL lse and
// Delta = rowsum(dO * O) (Appendix D), so on a kept block
//   P = exp(alpha q.k - lse_q)   (the global probabilities, no per-leaf renormalisation)
//   dP = dO V^T,   dS = P (dP - Delta_q)
//   dV += P^T dO,  dK += alpha dS^T Q,  dQ += alpha dS K           (IndexAdd)
// Two kernels per task, both reading Q/K/V/dO in place through TMA (no Gather copy):
//
//  bwd_dkdv: CTA = one 128-key tile of one key segment of one (b,h) plane.  K, V stay in smem; the
//    CTA loops over the 128-row query tiles of every query segment that keeps its key segment.
//    Per query tile, in two halves of 64 queries (so the elementwise pass of one half overlaps the
//    MMAs of the other):
//      S^T_h = K Q_h^T, dP^T_h = V dO_h^T          (tcgen05 SS, fp32 in TMEM)
//      P^T_h, dS^T_h  (bf16, written back into TMEM over S^T_h / dP^T_h by 4 warps, thread = key)
//      dV += P^T_h dO_h, dK += dS^T_h Q_h          (tcgen05 TS: A from TMEM, B = dO/Q MN-major)
//    Epilogue: dV, alpha dK read from TMEM and added into the fp32 accumulators.
//  bwd_dq:   CTA = one 128-query tile; loops over the key tiles of the kept key segments:
//      S_h = Q K_h^T, dP_h = dO V_h^T; dS_h (bf16 into TMEM); dQ += dS_h K_h (B = K MN-major).
//
// TMEM (512 columns): S 0..127 | dP 128..255 | acc0 256.. (dV or dQ) | acc1 256+D.. (dK).
// Warp roles (256 threads): 0 TMA producer, 1 MMA issuer (warp-wide, elected lane), 2 TMEM
// allocator, 3 idle, 4-7 elementwise + epilogue (thread = TMEM lane).
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "attn_common.cuh"
#include "task_params.cuh"

namespace cqs {

// Elementwise (EW) pass on 8 warps: warps w and w + 4 share a TMEM lane quarter (rows) and split
// each 64-column half-tile into 32-column chunks, so two warps per SM sub-partition feed the MUFU
// (one warp alone reaches ~79% of its rate, two ~89%: tools/softmax_bench.cu).  Each chunk's P / dS
// (bf16 pairs) is written at the start of its own 32 source columns, so the two warps never write
// columns the other still has to read; the MMAs read the A operand at ew_acol(kk).
constexpr bool kEW8 = true;
constexpr int kBwdThreads = kEW8 ? 384 : 256;
__device__ __forceinline__ constexpr uint32_t ew_ocol(int c) { return kEW8 ? c * 32 : c * 16; }
__device__ __forceinline__ constexpr uint32_t ew_acol(int kk) {
  return kEW8 ? (kk >> 1) * 32 + (kk & 1) * 8 : kk * 8;
}

template <int D>
struct BwdCfg {
  static constexpr int kBoxes = D / 64;
  static constexpr int kTile = 128 * D * 2;             // one 128-row bf16 tile
  static constexpr int kLdBytes = 2 * 128 * 4;          // -lse*log2e | Delta of 128 query rows
  static constexpr int kStages = D == 128 ? 2 : 4;
  static constexpr int kStageKV = 2 * kTile + kLdBytes; // dK/dV kernel stage: Q, dO, lse/Delta
  static constexpr int kSmemKV = 2 * kTile + kStages * kStageKV + 1024 + 256;
  static constexpr int kSmemQ = 2 * kTile + kStages * 2 * kTile + 1024 + 256;
  static constexpr uint32_t kColS = 0, kColP = 128, kColA0 = 256, kColA1 = 256 + D;
  // dQ kernel: the CTA's Q and dO tiles (the A operands of S = Q K^T and dP = dO V^T, fixed for the
  // whole CTA) live in the TMEM columns after the dQ accumulator, so those MMAs read only K / V
  // from shared memory (an SS MMA at M = 128, N = 64 needs 192 B/clk of SMEM, over the 128 B/clk
  // available; with A in TMEM it needs 64)
  static constexpr uint32_t kColQ = 256 + D, kColdO = 256 + D + D / 2;
  static constexpr bool kQdOInTmem = true;
  // dK/dV kernel at D = 64: the CTA's K and V tiles (A of S^T = K Q^T, dP^T = V dO^T) in TMEM after
  // the dK accumulator; at D = 128 the four 128-column regions use all 512 columns
  static constexpr uint32_t kColKT = 256 + 2 * D, kColVT = 256 + 2 * D + D / 2;
  static constexpr bool kKVInTmem = D == 64;
};

// descriptor offset of the 16-wide K step `ks` in a K-major SW128 tile of 128 rows
__device__ __forceinline__ uint64_t kstep_off(int ks) {
  return uint64_t(((ks >> 2) * (128 * 128) + (ks & 3) * 32) >> 4);
}

// One elementwise pass over 32 columns of S / dP held in TMEM (fp32 at tS / tP), writing P and dS
// as packed bf16 pairs to the 16 columns at oS / oP (chunk c of a 64-column half lands on columns
// ew_ocol(c).. of the half, the K-major TMEM A operand of the next MMA, read at ew_acol(kk)).  nl2/dl2: per-column
// (-lse*log2e, Delta) pairs; valid: columns >= valid are masked to zero.
template <bool kWriteP>
__device__ __forceinline__ void bwd_ew_chunk(uint32_t tS, uint32_t tP, uint32_t oS, uint32_t oP,
                                             int col0, int valid,
                                             uint64_t sc2, const uint64_t* nl2,
                                             const uint64_t* dl2, bool per_col) {
  uint32_t sv[32], dv[32];
  ptx::tmem_ld32(tS, sv);
  ptx::tmem_ld32(tP, dv);
  ptx::tmem_ld_wait();
  uint32_t pk[16], dk[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint64_t nl = per_col ? nl2[i] : nl2[0], dl = per_col ? dl2[i] : dl2[0];
    float x0, x1;
    ptx::f2_split(ptx::ffma2(ptx::f2(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])),
                             sc2, nl),
                  x0, x1);
    float p0 = ptx::ex2(x0), p1 = ptx::ex2(x1);
    if (col0 + 2 * i >= valid) p0 = 0.f;
    if (col0 + 2 * i + 1 >= valid) p1 = 0.f;
    const uint64_t pp = ptx::f2(p0, p1);
    const uint64_t t =
        ptx::fsub2(ptx::f2(__uint_as_float(dv[2 * i]), __uint_as_float(dv[2 * i + 1])), dl);
    float d0, d1;
    ptx::f2_split(ptx::fmul2(pp, t), d0, d1);
    if (kWriteP) pk[i] = ptx::pack_bf16(p0, p1);
    dk[i] = ptx::pack_bf16(d0, d1);
  }
  if (kWriteP) ptx::tmem_st16(oS, pk);
  ptx::tmem_st16(oP, dk);
}

// fp32 accumulator rows += scale * TMEM accumulator row (D columns starting at column tA)
template <int D>
__device__ __forceinline__ void bwd_store_acc(uint32_t tA, float* __restrict__ dst, float scale,
                                              bool live) {
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    uint32_t v[32];
    ptx::tmem_ld32(tA + c * 32, v);
    ptx::tmem_ld_wait();
    if (live) {
      float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 a = d4[i];
        a.x = fmaf(scale, __uint_as_float(v[4 * i + 0]), a.x);
        a.y = fmaf(scale, __uint_as_float(v[4 * i + 1]), a.y);
        a.z = fmaf(scale, __uint_as_float(v[4 * i + 2]), a.z);
        a.w = fmaf(scale, __uint_as_float(v[4 * i + 3]), a.w);
        d4[i] = a;
      }
    }
  }
}

// Work item of a launch: head-major rasterization like the forward (the CTAs in flight share the
// (b,h) plane and its streamed tiles in L2).  Returns the segment and the tile's row offset in it.
__device__ __forceinline__ void bwd_item(const TaskParams& tp, int& bh, int& seg, int& off) {
  bh = blockIdx.x / tp.n_items;
  const int item = blockIdx.x % tp.n_items;
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  seg = tp.order[oi];
  off = (item - (oi ? tp.item_end[oi - 1] : 0)) * 128;
}

// =============================================================================================
// dK / dV.  tp is the TRANSPOSED task descriptor: kept[b] bit a = query segment a keeps key
// segment b, items = 128-key tiles of key segments with at least one keeper.
// =============================================================================================
template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const __grid_constant__ TaskParams tp, const float* __restrict__ ld,
                    int64_t ld_pitch, int64_t n_rows, float* __restrict__ dk_acc, float* __restrict__ dv_acc, float scale_log2,
                    float scale) {
  using C = BwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::kTile;
  uint8_t* sStage = smem + 2 * C::kTile;          // [kStages][Q | dO | lse,Delta]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + C::kStages * C::kStageKV);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;
  uint64_t* qd_empty = qd_full + C::kStages;
  uint64_t* s_full = qd_empty + C::kStages;       // 2 (halves)
  uint64_t* p_full = s_full + 2;                  // 2
  uint64_t* acc_done = p_full + 2;
  uint64_t* kv_tm = acc_done + 1;                 // K / V copied into TMEM (kKVInTmem, 4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_tm + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bh, b, k_off;
  bwd_item(tp, bh, b, k_off);
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t qmask = tp.kept[b];
  int n_q = 0;
  for (uint32_t m = qmask; m; m &= m - 1) n_q += (tp.seg_len[__ffs(m) - 1] + 127) / 128;

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&qd_full[s], 1);
      ptx::mbar_init(&qd_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      ptx::mbar_init(&s_full[h], 1);
      ptx::mbar_init(&p_full[h], kEW8 ? 8 : 4);
    }
    ptx::mbar_init(acc_done, 1);
    ptx::mbar_init(kv_tm, 4);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // whole warp: lane 0 issues the TMA tiles, all 32 lanes copy the tile's (-lse*log2e, Delta)
    // rows (plain loads: a query tile starts at any row, too unaligned for a bulk copy)
    const int k_row = tp.seg_src[b] + k_off;
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmQ);
      ptx::tma_prefetch_desc(&tmdO);
      ptx::mbar_arrive_expect_tx(kv_full, 2 * C::kTile);
      for (int bx = 0; bx < C::kBoxes; ++bx) {
        ptx::tma_load_4d(sK + bx * 128 * 128, &tmK, kv_full, bx * 64, k_row, hi, bi);
        ptx::tma_load_4d(sV + bx * 128 * 128, &tmV, kv_full, bx * 64, k_row, hi, bi);
      }
    }
    const float* ld_plane = ld + int64_t(bh) * 2 * ld_pitch + (lane >> 4) * ld_pitch;
    KvCursor cq;
    cq.init(&tp, qmask);
    for (int i = 0; i < n_q; ++i) {
      const int s = i % C::kStages;
      ptx::mbar_wait(&qd_empty[s], ((i / C::kStages) & 1) ^ 1);
      uint8_t* st = sStage + s * C::kStageKV;
      const int q_row = cq.row();                                    // TMA (Q / dO) row
      const int g_row = tp.seg_dst[cq.seg] + cq.kt * 128;            // global row (lse / Delta)
      float* dst = reinterpret_cast<float*>(st + 2 * C::kTile) + (lane >> 4) * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = (lane & 15) + 16 * u;
        dst[r] = g_row + r < n_rows ? ld_plane[g_row + r] : 0.f;
      }
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&qd_full[s], 2 * C::kTile);
        for (int bx = 0; bx < C::kBoxes; ++bx) {
          ptx::tma_load_4d(st + bx * 128 * 128, &tmQ, &qd_full[s], bx * 64, q_row, hi, bi);
          ptx::tma_load_4d(st + C::kTile + bx * 128 * 128, &tmdO, &qd_full[s], bx * 64, q_row, hi,
                           bi);
        }
      }
      cq.next();
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 64, 0, 0);   // S^T half: 128 keys x 64 q
    constexpr uint32_t idesc_g = ptx::idesc_bf16(128, D, 0, 1);    // dV/dK: B = dO/Q MN-major
    const uint64_t dK = ptx::smem_desc_sw128(ptx::smem_u32(sK), 16, 1024);
    const uint64_t dV = ptx::smem_desc_sw128(ptx::smem_u32(sV), 16, 1024);
    const uint64_t dSt = ptx::smem_desc_sw128(ptx::smem_u32(sStage), 16, 1024);
    const uint64_t dStMN = ptx::smem_desc_sw128(ptx::smem_u32(sStage), 128 * 128, 1024);
    auto issue_SdP = [&](int i, int h) {
      const uint64_t st = uint64_t((i % C::kStages) * C::kStageKV) >> 4;
      const uint64_t hq = uint64_t(h * 64 * 128) >> 4;   // query rows h*64.. of the tile
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        if constexpr (C::kKVInTmem)
          ptx::mma_ts_elect(tmem + C::kColS + h * 64, tmem + C::kColKT + ks * 8,
                            dSt + st + hq + kstep_off(ks), idesc_s, ks > 0);
        else
          ptx::mma_ss_elect(tmem + C::kColS + h * 64, dK + kstep_off(ks),
                            dSt + st + hq + kstep_off(ks), idesc_s, ks > 0);
      }
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        if constexpr (C::kKVInTmem)
          ptx::mma_ts_elect(tmem + C::kColP + h * 64, tmem + C::kColVT + ks * 8,
                            dSt + st + (C::kTile >> 4) + hq + kstep_off(ks), idesc_s, ks > 0);
        else
          ptx::mma_ss_elect(tmem + C::kColP + h * 64, dV + kstep_off(ks),
                            dSt + st + (C::kTile >> 4) + hq + kstep_off(ks), idesc_s, ks > 0);
      }
      ptx::mma_commit_elect(&s_full[h]);
    };
    auto issue_G = [&](int i, int h) {
      const uint64_t st = uint64_t((i % C::kStages) * C::kStageKV) >> 4;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t qr = uint64_t((h * 64 + kk * 16) * 128) >> 4;
        const uint32_t acc = (i | h | kk) != 0;
        ptx::mma_ts_elect(tmem + C::kColA0, tmem + C::kColS + h * 64 + ew_acol(kk),
                          dStMN + st + (C::kTile >> 4) + qr, idesc_g, acc);   // dV += P^T dO
        ptx::mma_ts_elect(tmem + C::kColA1, tmem + C::kColP + h * 64 + ew_acol(kk),
                          dStMN + st + qr, idesc_g, acc);                       // dK += dS^T Q
      }
    };
    ptx::mbar_wait(C::kKVInTmem ? kv_tm : kv_full, 0);
    ptx::mbar_wait(&qd_full[0], 0);
    ptx::tc_fence_after();
    issue_SdP(0, 0);
    issue_SdP(0, 1);
    for (int i = 0; i < n_q; ++i) {
      const bool more = i + 1 < n_q;
      ptx::mbar_wait(&p_full[0], i & 1);
      ptx::tc_fence_after();
      issue_G(i, 0);
      if (more) {
        const int s1 = (i + 1) % C::kStages;
        ptx::mbar_wait(&qd_full[s1], ((i + 1) / C::kStages) & 1);
        ptx::tc_fence_after();
        issue_SdP(i + 1, 0);
      }
      ptx::mbar_wait(&p_full[1], i & 1);
      ptx::tc_fence_after();
      issue_G(i, 1);
      ptx::mma_commit_elect(&qd_empty[i % C::kStages]);
      if (more) issue_SdP(i + 1, 1);
    }
    ptx::mma_commit_elect(acc_done);
  } else if (warp >= 4) {
    const int sub = warp & 3;
    const int cw = (warp - 4) >> 2;                  // kEW8: this warp's 32-column chunk
    const int r = sub * 32 + lane;
    const uint32_t lane_base = uint32_t(sub * 32) << 16;
    const uint32_t tS = tmem + lane_base + C::kColS, tP = tmem + lane_base + C::kColP;
    const uint64_t sc2 = ptx::f2(scale_log2, scale_log2);
    if (C::kKVInTmem && cw == 0) {
      // key row r of K and V (one SW128 box at D = 64) -> TMEM columns kColKT / kColVT
      ptx::mbar_wait(kv_full, 0);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint8_t* base = (g ? sV : sK) + r * 128;
        uint32_t kv[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 u = *reinterpret_cast<const uint4*>(base + ((c ^ (r & 7)) << 4));
          kv[4 * c + 0] = u.x, kv[4 * c + 1] = u.y, kv[4 * c + 2] = u.z, kv[4 * c + 3] = u.w;
        }
        ptx::tmem_st32(tmem + lane_base + (g ? C::kColVT : C::kColKT), kv);
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(kv_tm);
    }
    KvCursor cq;
    cq.init(&tp, qmask);
    for (int i = 0; i < n_q; ++i) {
      const int valid_q = cq.valid();
      cq.next();
      const int s = i % C::kStages;
      ptx::mbar_wait(&qd_full[s], (i / C::kStages) & 1);   // lse/Delta visibility
      const float* sLD = reinterpret_cast<const float*>(sStage + s * C::kStageKV + 2 * C::kTile);
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        ptx::mbar_wait(&s_full[h], i & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < (kEW8 ? 1 : 2); ++cc) {
          const int c = kEW8 ? cw : cc;
          const int q0 = h * 64 + c * 32;
          bwd_ew_chunk<true>(tS + h * 64 + c * 32, tP + h * 64 + c * 32, tS + h * 64 + ew_ocol(c),
                             tP + h * 64 + ew_ocol(c), q0, valid_q, sc2,
                             reinterpret_cast<const uint64_t*>(sLD + q0),
                             reinterpret_cast<const uint64_t*>(sLD + 128 + q0), true);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[h]);
      }
    }
    ptx::mbar_wait(acc_done, 0);
    ptx::tc_fence_after();
    const bool live = r < min(128, tp.seg_len[b] - k_off);
    const int64_t idx = int64_t(tp.seg_dst[b] + k_off + r) * tp.BH + bh;
    if (!kEW8 || cw == 0) bwd_store_acc<D>(tmem + lane_base + C::kColA0, dv_acc + idx * D, 1.f, live);
    if (!kEW8 || cw == 1) bwd_store_acc<D>(tmem + lane_base + C::kColA1, dk_acc + idx * D, scale, live);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// =============================================================================================
// dQ.  tp is the forward task descriptor (items = 128-query tiles of active query segments).
// ld: [B*H][2][ld_pitch] fp32 (-lse*log2e, Delta).
// =============================================================================================
template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                  const __grid_constant__ TaskParams tp, const float* __restrict__ ld,
                  int64_t ld_pitch, int64_t n_rows, float* __restrict__ dq_acc, float scale_log2,
                  float scale) {
  using C = BwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + C::kTile;
  uint8_t* sStage = smem + 2 * C::kTile;          // [kStages][K | V]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + C::kStages * 2 * C::kTile);
  uint64_t* qd_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;
  uint64_t* p_full = s_full + 2;
  uint64_t* acc_done = p_full + 2;
  uint64_t* q_tm = acc_done + 1;                  // Q / dO copied into TMEM (4 EW warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_tm + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bh, a, q_off;
  bwd_item(tp, bh, a, q_off);
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t kmask = tp.kept[a];
  int n_kv = 0;
  for (uint32_t m = kmask; m; m &= m - 1) n_kv += (tp.seg_len[__ffs(m) - 1] + 127) / 128;

  if (threadIdx.x == 0) {
    ptx::mbar_init(qd_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      ptx::mbar_init(&s_full[h], 1);
      ptx::mbar_init(&p_full[h], kEW8 ? 8 : 4);
    }
    ptx::mbar_init(acc_done, 1);
    ptx::mbar_init(q_tm, 4);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmK);
      ptx::tma_prefetch_desc(&tmV);
      const int q_row = tp.seg_src[a] + q_off;
      ptx::mbar_arrive_expect_tx(qd_full, 2 * C::kTile);
      for (int bx = 0; bx < C::kBoxes; ++bx) {
        ptx::tma_load_4d(sQ + bx * 128 * 128, &tmQ, qd_full, bx * 64, q_row, hi, bi);
        ptx::tma_load_4d(sdO + bx * 128 * 128, &tmdO, qd_full, bx * 64, q_row, hi, bi);
      }
      KvCursor ck;
      ck.init(&tp, kmask);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % C::kStages;
        ptx::mbar_wait(&kv_empty[s], ((j / C::kStages) & 1) ^ 1);
        uint8_t* st = sStage + s * 2 * C::kTile;
        ptx::mbar_arrive_expect_tx(&kv_full[s], 2 * C::kTile);
        const int k_row = ck.row();
        for (int bx = 0; bx < C::kBoxes; ++bx) {
          ptx::tma_load_4d(st + bx * 128 * 128, &tmK, &kv_full[s], bx * 64, k_row, hi, bi);
          ptx::tma_load_4d(st + C::kTile + bx * 128 * 128, &tmV, &kv_full[s], bx * 64, k_row, hi,
                           bi);
        }
        ck.next();
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 64, 0, 0);   // S half: 128 q x 64 keys
    constexpr uint32_t idesc_g = ptx::idesc_bf16(128, D, 0, 1);    // dQ += dS K, K MN-major
    const uint64_t dQd = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 16, 1024);
    const uint64_t ddO = ptx::smem_desc_sw128(ptx::smem_u32(sdO), 16, 1024);
    const uint64_t dSt = ptx::smem_desc_sw128(ptx::smem_u32(sStage), 16, 1024);
    const uint64_t dStMN = ptx::smem_desc_sw128(ptx::smem_u32(sStage), 128 * 128, 1024);
    auto issue_SdP = [&](int j, int h) {
      const uint64_t st = uint64_t((j % C::kStages) * 2 * C::kTile) >> 4;
      const uint64_t hk = uint64_t(h * 64 * 128) >> 4;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        if constexpr (C::kQdOInTmem)
          ptx::mma_ts_elect(tmem + C::kColS + h * 64, tmem + C::kColQ + ks * 8,
                            dSt + st + hk + kstep_off(ks), idesc_s, ks > 0);
        else
          ptx::mma_ss_elect(tmem + C::kColS + h * 64, dQd + kstep_off(ks),
                            dSt + st + hk + kstep_off(ks), idesc_s, ks > 0);
      }
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        if constexpr (C::kQdOInTmem)
          ptx::mma_ts_elect(tmem + C::kColP + h * 64, tmem + C::kColdO + ks * 8,
                            dSt + st + (C::kTile >> 4) + hk + kstep_off(ks), idesc_s, ks > 0);
        else
          ptx::mma_ss_elect(tmem + C::kColP + h * 64, ddO + kstep_off(ks),
                            dSt + st + (C::kTile >> 4) + hk + kstep_off(ks), idesc_s, ks > 0);
      }
      ptx::mma_commit_elect(&s_full[h]);
    };
    auto issue_G = [&](int j, int h) {
      const uint64_t st = uint64_t((j % C::kStages) * 2 * C::kTile) >> 4;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t kr = uint64_t((h * 64 + kk * 16) * 128) >> 4;
        ptx::mma_ts_elect(tmem + C::kColA0, tmem + C::kColP + h * 64 + ew_acol(kk),
                          dStMN + st + kr, idesc_g, (j | h | kk) != 0);        // dQ += dS K
      }
    };
    ptx::mbar_wait(C::kQdOInTmem ? q_tm : qd_full, 0);
    ptx::mbar_wait(&kv_full[0], 0);
    ptx::tc_fence_after();
    issue_SdP(0, 0);
    issue_SdP(0, 1);
    for (int j = 0; j < n_kv; ++j) {
      const bool more = j + 1 < n_kv;
      ptx::mbar_wait(&p_full[0], j & 1);
      ptx::tc_fence_after();
      issue_G(j, 0);
      if (more) {
        const int s1 = (j + 1) % C::kStages;
        ptx::mbar_wait(&kv_full[s1], ((j + 1) / C::kStages) & 1);
        ptx::tc_fence_after();
        issue_SdP(j + 1, 0);
      }
      ptx::mbar_wait(&p_full[1], j & 1);
      ptx::tc_fence_after();
      issue_G(j, 1);
      ptx::mma_commit_elect(&kv_empty[j % C::kStages]);
      if (more) issue_SdP(j + 1, 1);
    }
    ptx::mma_commit_elect(acc_done);
  } else if (warp >= 4) {
    const int sub = warp & 3;
    const int cw = (warp - 4) >> 2;                  // kEW8: this warp's 32-column chunk
    const int r = sub * 32 + lane;
    const uint32_t lane_base = uint32_t(sub * 32) << 16;
    const uint32_t tS = tmem + lane_base + C::kColS, tP = tmem + lane_base + C::kColP;
    const uint64_t sc2 = ptx::f2(scale_log2, scale_log2);
    const int64_t q_row = tp.seg_dst[a] + q_off + r;   // global row of the lse / Delta tables
    float nl = 0.f, dl = 0.f;
    if (q_row < n_rows) {
      nl = ld[int64_t(bh) * 2 * ld_pitch + q_row];
      dl = ld[(int64_t(bh) * 2 + 1) * ld_pitch + q_row];
    }
    const uint64_t nl2 = ptx::f2(nl, nl), dl2 = ptx::f2(dl, dl);
    if (C::kQdOInTmem && cw == 0) {
      // row r of the Q and dO tiles (SW128 boxes of 64 columns: 16-byte chunk c of row r sits at
      // chunk c ^ (r & 7)) -> packed bf16 pairs -> TMEM columns kColQ / kColdO (packed like P)
      ptx::mbar_wait(qd_full, 0);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint8_t* base = (g ? sdO : sQ) + r * 128;
#pragma unroll
        for (int bx = 0; bx < C::kBoxes; ++bx) {
          uint32_t qv[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 u =
                *reinterpret_cast<const uint4*>(base + bx * 128 * 128 + ((c ^ (r & 7)) << 4));
            qv[4 * c + 0] = u.x, qv[4 * c + 1] = u.y, qv[4 * c + 2] = u.z, qv[4 * c + 3] = u.w;
          }
          ptx::tmem_st32(tmem + lane_base + (g ? C::kColdO : C::kColQ) + bx * 32, qv);
        }
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(q_tm);
    }
    KvCursor ck;
    ck.init(&tp, kmask);
    for (int j = 0; j < n_kv; ++j) {
      const int valid_k = ck.valid();
      ck.next();
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        ptx::mbar_wait(&s_full[h], j & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < (kEW8 ? 1 : 2); ++cc) {
          const int c = kEW8 ? cw : cc;
          bwd_ew_chunk<false>(tS + h * 64 + c * 32, tP + h * 64 + c * 32, tS + h * 64 + ew_ocol(c),
                              tP + h * 64 + ew_ocol(c), h * 64 + c * 32, valid_k, sc2, &nl2, &dl2,
                              false);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[h]);
      }
    }
    ptx::mbar_wait(acc_done, 0);
    ptx::tc_fence_after();
    const bool live = r < min(128, tp.seg_len[a] - q_off);
    const int64_t idx = int64_t(tp.seg_dst[a] + q_off + r) * tp.BH + bh;
    if (kEW8)   // each warp of the pair adds half of the D columns
      bwd_store_acc<D / 2>(tmem + lane_base + C::kColA0 + cw * (D / 2),
                           dq_acc + idx * D + cw * (D / 2), scale, live);
    else
      bwd_store_acc<D>(tmem + lane_base + C::kColA0, dq_acc + idx * D, scale, live);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Delta = rowsum(dO * O) and -lse*log2e, transposed to [B*H][2][ld_pitch] (query rows contiguous
// per plane, the layout the dK/dV kernel loads with one TMA box per query tile).  One thread per
// 8-element (16-byte) chunk of a row; D/8 lanes per row reduce with shuffles.
template <int D>
__global__ void __launch_bounds__(256)
    bwd_prep_kernel(const uint16_t* __restrict__ o, const uint16_t* __restrict__ dO,
                    int64_t sB, int64_t sH, int64_t sN, const float* __restrict__ lse,
                    int64_t lse_pitch, int B, int H, int64_t N, int64_t row0, int64_t ld_pitch,
                    float* __restrict__ ld) {
  constexpr int kLanes = D / 8;
  const int64_t rows = int64_t(B) * H * N;
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t row = g / kLanes;            // (bh, n) with n fastest
  const int ch = int(g % kLanes);
  float acc = 0.f;
  int64_t n = 0, bh = 0;
  if (row < rows) {
    bh = row / N;
    n = row - bh * N;
    const int64_t bb = bh / H, hh = bh - bb * H;
    const int64_t off = bb * sB + hh * sH + n * sN + ch * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(o + off);
    const uint4 d = *reinterpret_cast<const uint4*>(dO + off);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc = fmaf(__uint_as_float(av[i] << 16), __uint_as_float(dv[i] << 16), acc);
      acc = fmaf(__uint_as_float(av[i] & 0xffff0000u), __uint_as_float(dv[i] & 0xffff0000u), acc);
    }
  }
#pragma unroll
  for (int w = kLanes / 2; w > 0; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
  if (row < rows && ch == 0) {
    ld[bh * 2 * ld_pitch + row0 + n] = -lse[bh * lse_pitch + n] * 1.4426950408889634f;
    ld[(bh * 2 + 1) * ld_pitch + row0 + n] = acc;
  }
}

template <int D>
static cudaError_t launch_bwd_impl(const CUtensorMap* maps, const TaskParams& tpq,
                                   const TaskParams& tpk, const float* ld, int64_t ld_pitch,
                                   int64_t N, float* dq, float* dk, float* dv, float scale,
                                   cudaStream_t st) {
  static std::atomic<uint64_t> cfg_kv{0}, cfg_q{0};
  using C = BwdCfg<D>;
  cudaError_t e = set_smem_attr_once(bwd_dkdv_kernel<D>, C::kSmemKV, cfg_kv);
  if (e == cudaSuccess) e = set_smem_attr_once(bwd_dq_kernel<D>, C::kSmemQ, cfg_q);
  if (e != cudaSuccess) return e;
  const float sl2 = scale * 1.4426950408889634f;
  const int64_t gk = int64_t(tpk.n_items) * tpk.BH, gq = int64_t(tpq.n_items) * tpq.BH;
  if (gk > 0)
    bwd_dkdv_kernel<D><<<dim3(unsigned(gk)), kBwdThreads, C::kSmemKV, st>>>(
        maps[0], maps[1], maps[2], maps[3], tpk, ld, ld_pitch, N, dk, dv, sl2, scale);
  if (gq > 0)
    bwd_dq_kernel<D><<<dim3(unsigned(gq)), kBwdThreads, C::kSmemQ, st>>>(
        maps[0], maps[1], maps[2], maps[3], tpq, ld, ld_pitch, N, dq, sl2, scale);
  return cudaGetLastError();
}

// maps: Q, K, V, dO (bf16, 128-row boxes); ld: fp32 [BH][2][pitch] (-lse*log2e, Delta).
// The dK/dV + dQ kernel pair above.  A single fused kernel (tools/experiments/
// attn_bwd_fused_sm100.cu, not built; dQ by fp32 L2 reductions) was parity-green but 23% slower on B200 — its red.global traffic (64 KB per 128x128 block) saturates the per-SM L2
// reduction path (profiles/r01_notes.md).
cudaError_t launch_attn_bwd_bf16(int D, const CUtensorMap* maps, const TaskParams& tpq,
                                 const TaskParams& tpk, const float* ld, int64_t ld_pitch,
                                 int64_t N, float* dq, float* dk, float* dv, float scale,
                                 cudaStream_t st) {
  if (D == 128) return launch_bwd_impl<128>(maps, tpq, tpk, ld, ld_pitch, N, dq, dk, dv, scale, st);
  if (D == 64) return launch_bwd_impl<64>(maps, tpq, tpk, ld, ld_pitch, N, dq, dk, dv, scale, st);
  return cudaErrorInvalidValue;
}

// rows [row0, row0 + N) of the tables from O / dO rows 0..N of the given views (lse: [B*H][lse_pitch])
cudaError_t launch_bwd_prep(int D, const void* o, const void* dO, const int64_t* strides,
                            const float* lse, int64_t lse_pitch, int B, int H, int64_t N,
                            int64_t row0, int64_t ld_pitch, float* ld, cudaStream_t st) {
  const int64_t threads = int64_t(B) * H * N * (D / 8);
  const int64_t blocks = (threads + 255) / 256;
  if (blocks <= 0) return cudaSuccess;
  auto O = static_cast<const uint16_t*>(o);
  auto G = static_cast<const uint16_t*>(dO);
  if (D == 128)
    bwd_prep_kernel<128><<<unsigned(blocks), 256, 0, st>>>(O, G, strides[0], strides[1],
                                                           strides[2], lse, lse_pitch, B, H, N, row0, ld_pitch, ld);
  else if (D == 64)
    bwd_prep_kernel<64><<<unsigned(blocks), 256, 0, st>>>(O, G, strides[0], strides[1],
                                                          strides[2], lse, lse_pitch, B, H, N, row0, ld_pitch, ld);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace cqs

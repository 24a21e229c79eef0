// EXPERIMENT (built into libcqs, selected only by -DCQS_BWD_FUSED builds; the default backward is
// the dK/dV + dQ kernel pair in attn_bwd_sm100.cu, which measured 22% faster: 889 vs 1139 ms per
// C2 step with the vectorised dQ drain below, 1427 ms with one red.f32 per element
// (-DCQS_BWD_RED_SCALAR) — see profiles/r01_notes.md "Backward").
// Fused per-task CQS attention backward for D = 128 (sm_100a tcgen05 / TMEM / TMA): one kernel
// computes dK, dV AND dQ of a task (Algorithm 2), so S and dP are computed
// once per kept block (10·D FLOP per pair instead of the two-kernel split's 14·D).
//
// CTA = one 128-key tile (K, V resident in smem); it loops over the 128-row query tiles of every
// query segment that keeps the tile's key segment, in halves of 64 queries:
//   S^T_h = K Q_h^T, dP^T_h = V dO_h^T                       (SS MMAs -> TMEM, fp32)
//   EW (warps 4-7, thread = key): P^T = 2^(s·α·log2e − lse·log2e), dS^T = P^T (dP^T − Delta);
//       P^T (bf16) -> TMEM over S^T_h;  dS^T (bf16) -> smem sdS[h] (SW128, [key][64 q])
//   dV   += P^T_h dO_h        (TS: A = P^T in TMEM, B = dO MN-major)
//   dK   += dS^T_h Q_h        (SS: A = sdS K-major, B = Q MN-major)
//   dQ^T_h = K^T dS^T_h       (SS: A = K^T = sK read MN-major, B = sdS read MN-major; M = d = 128,
//                              N = 64 queries) into the TMEM columns of dP^T_h, which the EW pass
//                              has already consumed
//   drain (warps 8-11, thread = d = TMEM lane): tcgen05.ld the 64 columns, release the columns,
//       4x4 shuffle transposes within lane quads, then red.global.add.v4.f32 alpha·dQ into the fp32
//       dQ accumulator (a warp instruction covers 4 query rows x 32 consecutive d = 4 x 128 B)
// TMEM (512 columns): S^T | dP^T (= dQ^T after EW) | dV | dK.
// Shared memory: K, V (64 KB) + 2 stages x (Q, dO) (128 KB) + sdS[2] (32 KB) + lse/Delta (2 KB):
// 226 KB, so the dynamic smem base must already be 1024-byte aligned (checked; traps otherwise).
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "attn_common.cuh"
#include "task_params.cuh"

namespace cqs {

namespace fused {
constexpr int D = 128;
constexpr int kThreads = 384;
constexpr int kTile = 128 * D * 2;          // 32 KB
constexpr int kStages = 2;
constexpr int kOffK = 0, kOffV = kTile, kOffStage = 2 * kTile;       // stage: Q | dO
constexpr int kOffdS = kOffStage + kStages * 2 * kTile;              // [2][128 keys][128 B]
constexpr int kdSBytes = 128 * 128;
constexpr int kOffLD = kOffdS + 2 * kdSBytes;                        // [kStages][2][128] fp32
constexpr int kOffBar = kOffLD + kStages * 2 * 128 * 4;
constexpr int kSmem = kOffBar + 256;
constexpr uint32_t kColS = 0, kColP = 128, kColV = 256, kColK = 384;
static_assert(kSmem <= 232448, "fused backward smem budget");
}  // namespace fused

__device__ __forceinline__ uint64_t kstep_k(int ks) {   // K-major SW128 tile of 128 rows
  return uint64_t(((ks >> 2) * (128 * 128) + (ks & 3) * 32) >> 4);
}

__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__global__ void __launch_bounds__(fused::kThreads, 1)
    bwd_fused_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                     const __grid_constant__ TaskParams tp, const float* __restrict__ ld,
                     int64_t ld_pitch, int64_t n_rows, float* __restrict__ dq_acc,
                     float* __restrict__ dk_acc, float* __restrict__ dv_acc, float scale_log2,
                     float scale) {
  using namespace fused;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((ptx::smem_u32(smem) & 1023) != 0) __trap();   // SW128 operands need 1024-byte alignment
  uint8_t* sK = smem + kOffK;
  uint8_t* sV = smem + kOffV;
  uint8_t* sStage = smem + kOffStage;
  uint8_t* sdS = smem + kOffdS;
  float* sLD = reinterpret_cast<float*>(smem + kOffLD);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;             // kStages
  uint64_t* qd_empty = qd_full + kStages;   // kStages
  uint64_t* s_full = qd_empty + kStages;    // 2 halves
  uint64_t* p_full = s_full + 2;
  uint64_t* dq_full = p_full + 2;
  uint64_t* dq_empty = dq_full + 2;
  uint64_t* acc_done = dq_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x / tp.n_items, item = blockIdx.x % tp.n_items;
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  const int b = tp.order[oi];
  const int k_off = (item - (oi ? tp.item_end[oi - 1] : 0)) * 128;
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t qmask = tp.kept[b];
  int n_q = 0;
  for (uint32_t m = qmask; m; m &= m - 1) n_q += (tp.seg_len[__ffs(m) - 1] + 127) / 128;

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&qd_full[s], 1);
      ptx::mbar_init(&qd_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      ptx::mbar_init(&s_full[h], 1);
      ptx::mbar_init(&p_full[h], 4);
      ptx::mbar_init(&dq_full[h], 1);
      ptx::mbar_init(&dq_empty[h], 4);
    }
    ptx::mbar_init(acc_done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ============ producer: lane 0 TMA (K, V once; Q, dO per query tile), all lanes lse/Delta ====
    const int k_row = tp.seg_src[b] + k_off;
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmQ);
      ptx::tma_prefetch_desc(&tmdO);
      ptx::mbar_arrive_expect_tx(kv_full, 2 * kTile);
      for (int bx = 0; bx < 2; ++bx) {
        ptx::tma_load_4d(sK + bx * 128 * 128, &tmK, kv_full, bx * 64, k_row, hi, bi);
        ptx::tma_load_4d(sV + bx * 128 * 128, &tmV, kv_full, bx * 64, k_row, hi, bi);
      }
    }
    const float* ld_plane = ld + int64_t(bh) * 2 * ld_pitch + (lane >> 4) * ld_pitch;
    KvCursor cq;
    cq.init(&tp, qmask);
    for (int i = 0; i < n_q; ++i) {
      const int s = i % kStages;
      ptx::mbar_wait(&qd_empty[s], ((i / kStages) & 1) ^ 1);
      const int q_row = cq.row();
      const int g_row = tp.seg_dst[cq.seg] + cq.kt * 128;            // global row (lse / Delta)
      float* dst = sLD + s * 256 + (lane >> 4) * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = (lane & 15) + 16 * u;
        dst[r] = g_row + r < n_rows ? ld_plane[g_row + r] : 0.f;
      }
      __syncwarp();
      if (lane == 0) {
        uint8_t* st = sStage + s * 2 * kTile;
        ptx::mbar_arrive_expect_tx(&qd_full[s], 2 * kTile);
        for (int bx = 0; bx < 2; ++bx) {
          ptx::tma_load_4d(st + bx * 128 * 128, &tmQ, &qd_full[s], bx * 64, q_row, hi, bi);
          ptx::tma_load_4d(st + kTile + bx * 128 * 128, &tmdO, &qd_full[s], bx * 64, q_row, hi,
                           bi);
        }
      }
      cq.next();
    }
  } else if (warp == 1) {
    // ============ MMA issuer (whole warp; one elected lane issues) ============
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 64, 0, 0);    // S^T / dP^T half
    constexpr uint32_t idesc_g = ptx::idesc_bf16(128, D, 0, 1);     // dV, dK (B MN-major)
    constexpr uint32_t idesc_q = ptx::idesc_bf16(128, 64, 1, 1);    // dQ^T (A, B MN-major)
    const uint64_t dK = ptx::smem_desc_sw128(ptx::smem_u32(sK), 16, 1024);
    const uint64_t dV = ptx::smem_desc_sw128(ptx::smem_u32(sV), 16, 1024);
    const uint64_t dKmn = ptx::smem_desc_sw128(ptx::smem_u32(sK), 128 * 128, 1024);
    const uint64_t dSt = ptx::smem_desc_sw128(ptx::smem_u32(sStage), 16, 1024);
    const uint64_t dStMN = ptx::smem_desc_sw128(ptx::smem_u32(sStage), 128 * 128, 1024);
    const uint64_t ddS = ptx::smem_desc_sw128(ptx::smem_u32(sdS), 16, 1024);
    const uint64_t ddSmn = ptx::smem_desc_sw128(ptx::smem_u32(sdS), 128 * 128, 1024);
    auto stage_off = [](int i) { return uint64_t((i % kStages) * 2 * kTile) >> 4; };
    auto issue_S = [&](int i, int h) {
      const uint64_t st = stage_off(i), hq = uint64_t(h * 64 * 128) >> 4;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        ptx::mma_ss_elect(tmem + kColS + h * 64, dK + kstep_k(ks), dSt + st + hq + kstep_k(ks),
                          idesc_s, ks > 0);
    };
    auto issue_dP = [&](int i, int h) {
      const uint64_t st = stage_off(i), hq = uint64_t(h * 64 * 128) >> 4;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        ptx::mma_ss_elect(tmem + kColP + h * 64, dV + kstep_k(ks),
                          dSt + st + (kTile >> 4) + hq + kstep_k(ks), idesc_s, ks > 0);
      ptx::mma_commit_elect(&s_full[h]);
    };
    auto issue_G = [&](int i, int h) {
      const uint64_t st = stage_off(i);
      const uint64_t dsh = uint64_t(h * kdSBytes) >> 4;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {                 // K = this half's 64 queries
        const uint64_t qr = uint64_t((h * 64 + kk * 16) * 128) >> 4;
        const uint32_t acc = (i | h | kk) != 0;
        ptx::mma_ts_elect(tmem + kColV, tmem + kColS + h * 64 + kk * 8,
                          dStMN + st + (kTile >> 4) + qr, idesc_g, acc);        // dV += P^T dO
        ptx::mma_ss_elect(tmem + kColK, ddS + dsh + uint64_t(kk * 2), dStMN + st + qr, idesc_g,
                          acc);                                                  // dK += dS^T Q
      }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)                   // K = the tile's 128 keys
        ptx::mma_ss_elect(tmem + kColP + h * 64, dKmn + uint64_t((ks * 16 * 128) >> 4),
                          ddSmn + dsh + uint64_t((ks * 16 * 128) >> 4), idesc_q, ks > 0);
      ptx::mma_commit_elect(&dq_full[h]);
    };
    ptx::mbar_wait(kv_full, 0);
    ptx::mbar_wait(&qd_full[0], 0);
    ptx::tc_fence_after();
    for (int h = 0; h < 2; ++h) {
      issue_S(0, h);
      issue_dP(0, h);
    }
    for (int i = 0; i < n_q; ++i) {
      const bool more = i + 1 < n_q;
      for (int h = 0; h < 2; ++h) {
        ptx::mbar_wait(&p_full[h], i & 1);
        ptx::tc_fence_after();
        issue_G(i, h);
        if (h == 1) ptx::mma_commit_elect(&qd_empty[i % kStages]);
        if (more) {
          if (h == 0) {
            ptx::mbar_wait(&qd_full[(i + 1) % kStages], ((i + 1) / kStages) & 1);
            ptx::tc_fence_after();
          }
          issue_S(i + 1, h);
          ptx::mbar_wait(&dq_empty[h], i & 1);     // dQ^T_h drained: its columns are free
          ptx::tc_fence_after();
          issue_dP(i + 1, h);
        }
      }
    }
    ptx::mma_commit_elect(acc_done);
  } else if (warp >= 4 && warp < 8) {
    // ============ elementwise: P^T, dS^T (thread = key row = TMEM lane) + dK/dV epilogue ========
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t lane_base = uint32_t(sub * 32) << 16;
    const uint32_t tS = tmem + lane_base + kColS, tP = tmem + lane_base + kColP;
    const uint64_t sc2 = ptx::f2(scale_log2, scale_log2);
    // key rows past the segment hold other tokens: their dS^T must be zero or K^T dS^T would
    // leak them into dQ (their own dK / dV rows are simply not stored)
    const int valid_q_lim = r < min(128, tp.seg_len[b] - k_off) ? 128 : 0;
    KvCursor cq;
    cq.init(&tp, qmask);
    for (int i = 0; i < n_q; ++i) {
      const int valid_q = min(cq.valid(), valid_q_lim);
      cq.next();
      const int s = i % kStages;
      ptx::mbar_wait(&qd_full[s], (i / kStages) & 1);    // lse/Delta of this stage visible
      const float* ldq = sLD + s * 256;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        ptx::mbar_wait(&s_full[h], i & 1);
        ptx::tc_fence_after();
        uint8_t* drow = sdS + h * kdSBytes + r * 128;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int q0 = h * 64 + c * 32;
          uint32_t sv[32], dv[32];
          ptx::tmem_ld32(tS + h * 64 + c * 32, sv);
          ptx::tmem_ld32(tP + h * 64 + c * 32, dv);
          ptx::tmem_ld_wait();
          const uint64_t* nl2 = reinterpret_cast<const uint64_t*>(ldq + q0);
          const uint64_t* dl2 = reinterpret_cast<const uint64_t*>(ldq + 128 + q0);
          uint32_t pk[16], dk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float x0, x1;
            ptx::f2_split(ptx::ffma2(ptx::f2(__uint_as_float(sv[2 * j]),
                                             __uint_as_float(sv[2 * j + 1])), sc2, nl2[j]),
                          x0, x1);
            float p0 = ptx::ex2(x0), p1 = ptx::ex2(x1);
            if (q0 + 2 * j >= valid_q) p0 = 0.f;
            if (q0 + 2 * j + 1 >= valid_q) p1 = 0.f;
            const uint64_t t = ptx::fsub2(
                ptx::f2(__uint_as_float(dv[2 * j]), __uint_as_float(dv[2 * j + 1])), dl2[j]);
            float d0, d1;
            ptx::f2_split(ptx::fmul2(ptx::f2(p0, p1), t), d0, d1);
            pk[j] = ptx::pack_bf16(p0, p1);
            dk[j] = ptx::pack_bf16(d0, d1);
          }
          ptx::tmem_st16(tS + h * 64 + c * 16, pk);
          // dS^T row r, queries c*32 .. c*32+31 = 16-byte chunks c*4 .. c*4+3 of the 128-byte
          // row, SW128-swizzled (chunk ^ (row & 7))
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int chunk = (c * 4 + u) ^ (r & 7);
            *reinterpret_cast<uint4*>(drow + chunk * 16) =
                make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
          }
        }
        fence_proxy_async_smem();      // dS^T smem writes -> visible to the tensor core
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
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {
      float* dst = (g ? dk_acc : dv_acc) + idx * D;
      const float sc = g ? scale : 1.f;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(tmem + lane_base + (g ? kColK : kColV) + c * 32, v);
        ptx::tmem_ld_wait();
        if (live) {
          float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float4 a = d4[e];
            a.x = fmaf(sc, __uint_as_float(v[4 * e + 0]), a.x);
            a.y = fmaf(sc, __uint_as_float(v[4 * e + 1]), a.y);
            a.z = fmaf(sc, __uint_as_float(v[4 * e + 2]), a.z);
            a.w = fmaf(sc, __uint_as_float(v[4 * e + 3]), a.w);
            d4[e] = a;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ============ dQ drain (thread = d = TMEM lane): TMEM -> fp32 reductions in L2 ============
    const int sub = warp & 3;
    const int d = sub * 32 + lane;
    const uint32_t tQ = tmem + (uint32_t(sub * 32) << 16) + kColP;
    KvCursor cq;
    cq.init(&tp, qmask);
    for (int i = 0; i < n_q; ++i) {
      const int valid_q = cq.valid();
      const int64_t q_dst = int64_t(tp.seg_dst[cq.seg]) + int64_t(cq.kt) * 128;
      cq.next();
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        ptx::mbar_wait(&dq_full[h], i & 1);
        ptx::tc_fence_after();
        uint32_t v[64];
        ptx::tmem_ld32(tQ + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        ptx::tmem_ld32(tQ + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&dq_empty[h]);
        const int nv = min(64, valid_q - h * 64);
        const int64_t row_stride = int64_t(tp.BH) * D;
#ifdef CQS_BWD_RED_SCALAR
        float* base = dq_acc + (q_dst + h * 64) * tp.BH * D + int64_t(bh) * D + d;
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (j < nv) red_add_f32(base + j * row_stride, scale * __uint_as_float(v[j]));
#else
        // 4x4 transposes across lane quads (lane 4g+i holds d = 32 sub + 4g + i): afterwards lane
        // 4g+i holds, for query 4qb+i, the four consecutive d = 32 sub + 4g .. +3, so one
        // red.global.add.v4.f32 per (thread, 4 queries) and a warp instruction covers 4 query rows
        // x 128 B (4x fewer reduction instructions than one f32 per element)
        const int i4 = lane & 3;
        float* base = dq_acc + (q_dst + h * 64 + i4) * row_stride + int64_t(bh) * D + sub * 32 +
                      (lane & ~3);
#pragma unroll
        for (int qb = 0; qb < 16; ++qb) {
          float a0 = __uint_as_float(v[4 * qb]), a1 = __uint_as_float(v[4 * qb + 1]);
          float a2 = __uint_as_float(v[4 * qb + 2]), a3 = __uint_as_float(v[4 * qb + 3]);
          const bool lo2 = (i4 & 2) == 0, even = (i4 & 1) == 0;
          const float t0 = __shfl_xor_sync(0xffffffffu, lo2 ? a2 : a0, 2);
          const float t1 = __shfl_xor_sync(0xffffffffu, lo2 ? a3 : a1, 2);
          if (lo2) a2 = t0, a3 = t1;
          else a0 = t0, a1 = t1;
          const float u0 = __shfl_xor_sync(0xffffffffu, even ? a1 : a0, 1);
          const float u1 = __shfl_xor_sync(0xffffffffu, even ? a3 : a2, 1);
          if (even) a1 = u0, a3 = u1;
          else a0 = u0, a2 = u1;
          if (4 * qb + i4 < nv)
            red_add_v4(base + int64_t(4 * qb) * row_stride, scale * a0, scale * a1, scale * a2,
                       scale * a3);
        }
#endif
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// tp: the TRANSPOSED task descriptor (items = 128-key tiles; kept[b] = query segments keeping b).
cudaError_t launch_attn_bwd_fused(const CUtensorMap* maps, const TaskParams& tp, const float* ld,
                                  int64_t ld_pitch, int64_t N, float* dq, float* dk, float* dv,
                                  float scale, cudaStream_t st) {
  static std::atomic<uint64_t> cfg{0};
  cudaError_t e = set_smem_attr_once(bwd_fused_kernel, fused::kSmem, cfg);
  if (e != cudaSuccess) return e;
  const int64_t grid = int64_t(tp.n_items) * tp.BH;
  if (grid <= 0) return cudaSuccess;
  bwd_fused_kernel<<<dim3(unsigned(grid)), fused::kThreads, fused::kSmem, st>>>(
      maps[0], maps[1], maps[2], maps[3], tp, ld, ld_pitch, N, dq, dk, dv,
      scale * 1.4426950408889634f, scale);
  return cudaGetLastError();
}

}  // namespace cqs

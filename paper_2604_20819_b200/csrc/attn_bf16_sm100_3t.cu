// Per-task CQS attention kernel for D = 64: THREE 128-row query tiles per CTA, 96-key KV tiles.
//
// Same math and contract as attn_bf16_sm100.cu (Eq. 2 partial in FA form, P:43 / P:240, merged
// into the fp32 accumulator in the epilogue, Eq. 3).  At D = 64 a (q, k) pair carries
// 4·64 = 256 MMA FLOP and one exponential, so the softmax pass (MUFU.EX2 at 16 / clk / SM plus the
// in-order FFMA2 / FADD2 / F2FP stream around it), not the tensor core, bounds the kernel.  With
// two tiles per CTA each tile's loop is pass + (P·V + next S on the tensor core), and whenever one
// tile waits for its MMAs only one warp per SM sub-partition is issuing exponentials.  Three tiles
// keep two to three exp passes in flight per sub-partition while the third tile's MMAs run.
// TMEM (512 columns) holds S_t (96 fp32 columns; P written back over it as 48 packed bf16 columns)
// and O_t (64) for t = 0..2: 3 x 160 = 480 columns — hence 96-key tiles (3 x (128 + 64) = 576 would
// not fit).
//
// CTA = three 128-row tiles of one query segment (384 rows) of one (b,h) plane; warps:
//   warp 0      TMA producer (Q once, then K/V tiles through a kStages ring)
//   warp 1      MMA issuer: S_0(t) for all t, then per KV step j and tile t: PV_j(t), S_{j+1}(t)
//   warp 2      TMEM allocator
//   warps 4-15  softmax + correction + epilogue, tile t = warps 4 + 4t .. 7 + 4t (thread = row)
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "ptx.cuh"
#include "task_params.cuh"

namespace cqs {

namespace t3 {
constexpr int D = 64;
#ifndef CQS_T3_TILES
#define CQS_T3_TILES 3
#define CQS_T3_BN 96
#endif
constexpr int kTiles = CQS_T3_TILES;
constexpr int kBN3 = CQS_T3_BN;                        // keys per KV tile
constexpr int kThreads = 32 * (4 + 4 * kTiles);        // 512
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;   // 128
constexpr int kQBytes = kBM * D * 2;                   // 16 KB per tile (one SW128 box)
constexpr int kKVBytes = kBN3 * D * 2;                 // 12 KB per K or V tile
#ifndef CQS_T3_STAGES
#define CQS_T3_STAGES ((232448 - 2048 - kTiles * kQBytes) / kKVBytes)
#endif
constexpr int kStages = CQS_T3_STAGES;
constexpr int kSmemBytes = kTiles * kQBytes + kStages * kKVBytes + 1024 + 512;
static_assert(kSmemBytes <= 232448, "shared memory");
constexpr uint32_t kColS = 0;                          // S_t at 96 t
constexpr uint32_t kColO = kTiles * kBN3;              // O_t at 288 + 64 t
static_assert(kColO + kTiles * D <= 512, "TMEM columns");
// Rescale guard of the speculative pass (attn_bf16_sm100.cu): a row is rescaled (exact max, O and
// l scaled, pass redone) only when its P row sum against the running max exceeds kSumLimit.
constexpr float kSumLimit = 65536.0f;
// setmaxnreg split of the 512 x 128 launch registers: 4 producer / MMA / allocator warps at LO,
// 12 softmax warps at HI, with 128 (128 - LO) = 384 (HI - 128) (an unbalanced .inc blocks forever)
// (80 / 144 measured +1.5% over 56 / 152: fewer MMA-warp spills, none in the exp pass)
#ifndef CQS_T3_REG_LO
#define CQS_T3_REG_LO 80
#define CQS_T3_REG_HI 144
#endif
static_assert(128 * (kLaunchRegs - CQS_T3_REG_LO) == 128 * kTiles * (CQS_T3_REG_HI - kLaunchRegs),
              "register split");
// key pairs (i mod 8) whose exp2 runs as an FMA-pipe polynomial instead of MUFU.EX2
#ifndef CQS_T3_POLY_MASK
#define CQS_T3_POLY_MASK 0x0
#endif
constexpr uint32_t kPolyMask = CQS_T3_POLY_MASK;
#ifndef CQS_T3_ANYORDER
#define CQS_T3_ANYORDER 1
#endif
constexpr bool kAnyOrder = CQS_T3_ANYORDER != 0;
}  // namespace t3

__global__ void __launch_bounds__(t3::kThreads, 1)
    attn_bf16_sm100_3t_kernel(const __grid_constant__ CUtensorMap tmQ,   // box 64 x 128
                              const __grid_constant__ CUtensorMap tmK,   // box 64 x 96
                              const __grid_constant__ CUtensorMap tmV,   // box 64 x 96
                              const __grid_constant__ TaskParams tp, float* __restrict__ acc_o,
                              float* __restrict__ acc_lse, float scale_log2) {
  using namespace t3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                                  // [3][128 rows][128 B]
  uint8_t* sKV = smem + kTiles * kQBytes;              // [kStages][96 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kKVBytes);
  uint64_t* q_full = bars;                             // 1 (+ drain phase)
  uint64_t* kv_full = bars + 1;                        // kStages
  uint64_t* kv_empty = kv_full + kStages;              // kStages
  uint64_t* s_full = kv_empty + kStages;               // kTiles
  uint64_t* p_full = s_full + kTiles;                  // kTiles
  uint64_t* o_bar = p_full + kTiles;                   // kTiles
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + kTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work item: (query segment, kTiles x 128-row block) x (b,h) plane, head-major ----
  const int bh = blockIdx.x / tp.n_items, item = blockIdx.x % tp.n_items;
  int oi = 0;
  while (item >= tp.item_end[oi]) ++oi;
  const int a = tp.order[oi];
  const int q_off = (item - (oi ? tp.item_end[oi - 1] : 0)) * (kTiles * kBM);
  const int len_a = tp.seg_len[a];
  const int ntile = min(kTiles, (len_a - q_off + kBM - 1) / kBM);   // tiles with rows
  const int bi = bh / tp.H, hi = bh % tp.H;
  const uint32_t kmask = tp.kept[a];
  int n_kv = 0;
  for (uint32_t m = kmask; m; m &= m - 1) n_kv += (tp.seg_len[__ffs(m) - 1] + kBN3 - 1) / kBN3;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < kTiles; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 4);
      ptx::mbar_init(&o_bar[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CQS_T3_REG_LO) : "memory");
    if (warp == 0 && lane == 0) {
      // ================= TMA producer =================
      ptx::tma_prefetch_desc(&tmQ);
      ptx::tma_prefetch_desc(&tmK);
      ptx::tma_prefetch_desc(&tmV);
      const int q_row = tp.seg_src[a] + q_off;
      ptx::mbar_arrive_expect_tx(q_full, ntile * kQBytes);
      for (int t = 0; t < ntile; ++t)
        ptx::tma_load_4d(sQ + t * kQBytes, &tmQ, q_full, 0, q_row + t * kBM, hi, bi);
      int it = 0;
      auto load = [&](const CUtensorMap* map, int row) {
        const int s = it % kStages;
        ptx::mbar_wait(&kv_empty[s], ((it / kStages) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[s], kKVBytes);
        ptx::tma_load_4d(sKV + s * kKVBytes, map, &kv_full[s], 0, row, hi, bi);
        ++it;
      };
      KvCursorT<kBN3> ck, cv;
      ck.init(&tp, kmask);
      cv.init(&tp, kmask);
      load(&tmK, ck.row());   // stage order = MMA order: K_0, then per j: K_{j+1}, V_j
      ck.next();
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          load(&tmK, ck.row());
          ck.next();
        }
        load(&tmV, cv.row());
        cv.next();
      }
    } else if (warp == 1) {
      // ================= MMA issuer (whole warp, one elected lane issues) =================
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(kBM, kBN3, 0, 0);   // M=128, N=96
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(kBM, D, 0, 1);      // M=128, N=64
      const uint64_t dq0 = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 16, 1024);
      const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), 16, 1024);
      const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(sKV), kBN3 * 128, 1024);
      auto issue_S = [&](int t, int s) {   // S_t = Q_t K^T, K = D = 64 (4 K-steps of 32 bytes)
        const uint64_t qa = dq0 + uint64_t((t * kQBytes) >> 4);
        const uint64_t kb = dkv0 + uint64_t((s * kKVBytes) >> 4);
        const uint32_t d = tmem + kColS + uint32_t(t * kBN3);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          ptx::mma_ss_elect(d, qa + uint64_t(ks * 2), kb + uint64_t(ks * 2), idesc_qk, ks > 0);
        ptx::mma_commit_elect(&s_full[t]);
      };
      auto issue_PV = [&](int t, int s, bool acc) {   // O_t += P_t V, K = 96 keys (6 K-steps)
        const uint64_t vb = dv0 + uint64_t((s * kKVBytes) >> 4);
        const uint32_t d = tmem + kColO + uint32_t(t * D), pa = tmem + kColS + uint32_t(t * kBN3);
#pragma unroll
        for (int ks = 0; ks < kBN3 / 16; ++ks)
          ptx::mma_ts_elect(d, pa + ks * 8, vb + uint64_t((ks * 16 * 128) >> 4), idesc_pv,
                            (acc || ks > 0));
        ptx::mma_commit_elect(&o_bar[t]);
      };
      int it = 0;
      ptx::mbar_wait(q_full, 0);
      const int sK0 = it % kStages;
      ptx::mbar_wait(&kv_full[sK0], (it / kStages) & 1);
      ++it;
      ptx::tc_fence_after();
      for (int t = 0; t < ntile; ++t) issue_S(t, sK0);
      ptx::mma_commit_elect(&kv_empty[sK0]);
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
        if (kAnyOrder) {
          // serve the tiles in the order their P becomes ready (polling), not strictly 0, 1, 2
          uint32_t pending = (1u << ntile) - 1;
          while (pending) {
#pragma unroll
            for (int t = 0; t < kTiles; ++t) {
              if (!((pending >> t) & 1) || !ptx::mbar_try_wait(&p_full[t], j & 1)) continue;
              pending &= ~(1u << t);
              ptx::tc_fence_after();
              issue_PV(t, sV, j > 0);
              if (sKn >= 0) issue_S(t, sKn);
            }
          }
        } else {
          for (int t = 0; t < ntile; ++t) {
            ptx::mbar_wait(&p_full[t], j & 1);
            ptx::tc_fence_after();
            issue_PV(t, sV, j > 0);
            if (sKn >= 0) issue_S(t, sKn);
          }
        }
        ptx::mma_commit_elect(&kv_empty[sV]);
        if (sKn >= 0) ptx::mma_commit_elect(&kv_empty[sKn]);
      }
      ptx::mma_commit_elect(q_full);   // drain: all MMAs of this CTA retired
      ptx::mbar_wait(q_full, 1);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CQS_T3_REG_HI) : "memory");
    // ================= softmax / correction / epilogue =================
    const int t = (warp - 4) >> 2;
    if (t < ntile) {
      const int sub = warp & 3;
      const int r = sub * 32 + lane;
      const uint32_t lane_base = uint32_t(sub * 32) << 16;
      const uint32_t tS = tmem + lane_base + kColS + uint32_t(t * kBN3);
      const uint32_t tO = tmem + lane_base + kColO + uint32_t(t * D);
      const uint32_t a_sfull = ptx::smem_u32(&s_full[t]), a_pfull = ptx::smem_u32(&p_full[t]);
      float m = -INFINITY, l = 0.f;
      KvCursorT<kBN3> cur;
      cur.init(&tp, kmask);
      for (int j = 0; j < n_kv; ++j) {
        const int valid = cur.valid();
        cur.next();
        ptx::mbar_wait_a(a_sfull, j & 1);
        ptx::tc_fence_after();
        uint32_t sr[kBN3];
#pragma unroll
        for (int c = 0; c < kBN3 / 32; ++c)
          ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        ptx::tmem_ld_wait();
        float* s = reinterpret_cast<float*>(sr);
        if (valid < kBN3) {
#pragma unroll
          for (int c = 0; c < kBN3; ++c)
            if (c >= valid) s[c] = -INFINITY;
        }
        // one exp2 pass: p = 2^(s*scale_log2 - m_use) (packed FFMA2 argument, MUFU.EX2) fused per
        // 32-key chunk with the packed row sum, the bf16 pack and the tcgen05.st of P over S
        auto exp_pass = [&](float m_use) -> float {
          const uint64_t sc2 = ptx::f2(scale_log2, scale_log2), nm2 = ptx::f2(-m_use, -m_use);
          uint64_t rs2[4] = {0, 0, 0, 0};
#pragma unroll
          for (int c = 0; c < kBN3 / 32; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int ii = 0; ii < 16; ++ii) {
              const int i = 16 * c + ii;
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
          const uint64_t rr = ptx::fadd2(ptx::fadd2(rs2[0], rs2[1]), ptx::fadd2(rs2[2], rs2[3]));
          float a0, a1;
          ptx::f2_split(rr, a0, a1);
          return a0 + a1;
        };
        auto row_max = [&]() {   // exact raw row max of the tile (4 FMNMX chains, then a tree)
          float mx4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) mx4[u] = s[u];
#pragma unroll
          for (int c = 4; c < kBN3; c += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) mx4[u] = fmaxf(mx4[u], s[c + u]);
          }
          return fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        };
        float rowsum;
        if (j == 0) {
          m = row_max() * scale_log2;   // first tile: exact row max first
          rowsum = exp_pass(m);
        } else {
          // speculative pass against the running max m; only a row whose P sum shows a large p
          // (rare after the first tiles) is rescaled to its exact max and the pass redone
          rowsum = exp_pass(m);
          const bool need = !(rowsum <= kSumLimit);   // also catches inf
          if (__any_sync(0xffffffffu, need)) {
            const float m_new = need ? fmaxf(m, row_max() * scale_log2) : m;
            const float f = ptx::ex2(m - m_new);
            ptx::tmem_st_wait();
            ptx::mbar_wait(&o_bar[t], (j - 1) & 1);   // O must hold PV_{j-1}
            ptx::tc_fence_after();
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
            rowsum = exp_pass(m);
          }
        }
        l += rowsum;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_a(a_pfull);
      }
      // ---- epilogue: O_i = O / l, lse_i = ln(sum exp) -> merge into the accumulator ----
      ptx::mbar_wait(&o_bar[t], (n_kv - 1) & 1);
      ptx::tc_fence_after();
      const int row_in_seg = q_off + t * kBM + r;
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
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

cudaError_t launch_attn_bf16_3t(const CUtensorMap* maps, const TaskParams& tp, float* acc_o,
                                float* acc_lse, float scale, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = set_smem_attr_once(attn_bf16_sm100_3t_kernel, t3::kSmemBytes, configured);
  if (e != cudaSuccess) return e;
  const int64_t grid = int64_t(tp.n_items) * tp.BH;
  if (grid <= 0) return cudaSuccess;
  attn_bf16_sm100_3t_kernel<<<dim3(unsigned(grid)), t3::kThreads, t3::kSmemBytes, stream>>>(
      maps[0], maps[1], maps[2], tp, acc_o, acc_lse, scale * 1.4426950408889634f);
  return cudaGetLastError();
}

}  // namespace cqs

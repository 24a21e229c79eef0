// LSE merge / finalize kernels (Eq. 3 in LSE form, PAPER.md P:48-52 with Den_j = exp(lse_j),
// Num_j = O_j Den_j).  HBM-bound: flat 16-byte vector loads of the D-contiguous fp32 rows,
// coalesced across the warp, several loads in flight per thread; bf16/fp32 output cast fused.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "cqs_internal.h"

namespace cqs {

constexpr int kMaxMergeParts = 16;

struct MergeParts {
  int32_t n;
  const float* o[kMaxMergeParts];
  const float* l[kMaxMergeParts];
};

__global__ void fill_f32_kernel(float* __restrict__ p, int64_t n, float val) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = val;
}

__device__ __forceinline__ void store4(float* dst, float4 v) { *reinterpret_cast<float4*>(dst) = v; }
__device__ __forceinline__ void store4(__nv_bfloat16* dst, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst) = u;
}


__device__ __forceinline__ float fast_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Eq. 3 weights of one unit in base 2 (MUFU ex2 / lg2: the accurate expf / logf and the 64-bit
// index divisions of the first version ran on the XU pipe and held the R = 8 merge at 70% of HBM
// bandwidth).  NP = the parts this instantiation supports (a power of two >= parts.n).
template <int NP>
__device__ __forceinline__ void unit_weights(const MergeParts& parts, const float* acc_lse,
                                             int64_t unit, float (&w)[NP + 1], float& lse) {
  constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.69314718055994531f;
  const float la = acc_lse ? acc_lse[unit] : -INFINITY;
  float mx = la;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    w[j] = j < parts.n ? parts.l[j][unit] : -INFINITY;
    mx = fmaxf(mx, w[j]);
  }
  if (mx == -INFINITY) {
#pragma unroll
    for (int j = 0; j <= NP; ++j) w[j] = 0.f;
    lse = -INFINITY;
    return;
  }
  const float mb = mx * kLog2e;
  // exp(l - mx) = 2^(l log2e - mx log2e); -inf entries give 2^-inf = 0
  w[NP] = fast_ex2(fmaf(la, kLog2e, -mb));
  float s = w[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    w[j] = fast_ex2(fmaf(w[j], kLog2e, -mb));
    s += w[j];
  }
  const float inv = 1.f / s;
#pragma unroll
  for (int j = 0; j <= NP; ++j) w[j] *= inv;
  lse = mx + fast_lg2(s) * kLn2;
}

// One unit = one (row, plane) of D fp32 values.  min(32, D/4) lanes share a unit (one float4
// column each, looping when D/4 > 32), so a warp covers 32 / lanes units per step; each lane
// takes U units per iteration (U = 8 / (NP + 1) rounded down, >= 1) and issues all their
// U x (NP + 1) 16-byte loads back to back, so even a 1-part merge keeps several loads in flight.
// The weights are recomputed by each lane of a unit from broadcast lse loads.
template <typename OutT, int NP, typename Idx>
__global__ void __launch_bounds__(256)
    merge_kernel(Idx nunits, int BH, int H, int D4, MergeParts parts, float* __restrict__ acc_o,
                 float* __restrict__ acc_lse, bool acc_write, OutT* __restrict__ out, int64_t sB,
                 int64_t sH, int64_t sN, int64_t out_row0, int64_t n_total,
                 float* __restrict__ lse_out) {
  constexpr int U = 8 / (NP + 1) > 1 ? 8 / (NP + 1) : 1;
  const int lane = threadIdx.x & 31;
  const int lpu = D4 < 32 ? D4 : 32, upw = 32 / lpu;
  const int lu = lane / lpu, sub = lane - lu * lpu;
  if (lu >= upw) return;
  const Idx warp0 = Idx((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5);
  const Idx nwarps = Idx((int64_t(gridDim.x) * blockDim.x) >> 5);
  const Idx gstep = Idx(upw) * U;
  for (Idx g = warp0 * gstep; g < nunits; g += nwarps * gstep) {
    float w[U][NP + 1];
    float lse[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const Idx unit = g + Idx(i * upw + lu);
      if (unit < nunits) unit_weights<NP>(parts, acc_lse, int64_t(unit), w[i], lse[i]);
    }
    for (int d4 = sub; d4 < D4; d4 += lpu) {
      float4 x[U][NP + 1];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const Idx unit = g + Idx(i * upw + lu);
        if (unit >= nunits) continue;
        const int64_t f = int64_t(unit) * D4 + d4;
#pragma unroll
        for (int j = 0; j < NP; ++j)
          if (w[i][j] != 0.f) x[i][j] = reinterpret_cast<const float4*>(parts.o[j])[f];
        if (w[i][NP] != 0.f) x[i][NP] = reinterpret_cast<const float4*>(acc_o)[f];
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const Idx unit = g + Idx(i * upw + lu);
        if (unit >= nunits) continue;
        const int64_t f = int64_t(unit) * D4 + d4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j <= NP; ++j) {
          if (w[i][j] == 0.f) continue;
          v.x = fmaf(w[i][j], x[i][j].x, v.x);
          v.y = fmaf(w[i][j], x[i][j].y, v.y);
          v.z = fmaf(w[i][j], x[i][j].z, v.z);
          v.w = fmaf(w[i][j], x[i][j].w, v.w);
        }
        if (acc_write) reinterpret_cast<float4*>(acc_o)[f] = v;
        if (out) {
          const Idx r = unit / Idx(BH);
          const int p = int(unit - r * Idx(BH));
          const int bb = p / H, hh = p - bb * H;
          store4(out + int64_t(bb) * sB + int64_t(hh) * sH + (out_row0 + int64_t(r)) * sN + 4 * d4,
                 v);
        }
      }
    }
    if (sub == 0) {
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const Idx unit = g + Idx(i * upw + lu);
        if (unit >= nunits) continue;
        if (acc_write) acc_lse[unit] = lse[i];
        if (lse_out) {
          const Idx r = unit / Idx(BH);
          const int p = int(unit - r * Idx(BH));
          lse_out[int64_t(p) * n_total + out_row0 + int64_t(r)] = lse[i];
        }
      }
    }
  }
}

// Finalize (no parts): O = acc_o (0 where acc_lse = -inf; acc_lse may be NULL), lse = acc_lse; a pure streaming
// copy + cast.  Thread -> (unit, float4 column) with D4 = D/4 a power of two (shift), 32-bit index
// math when the unit count fits (the 64-bit divisions of a flat int64 index ran on the XU pipe
// and held this kernel at 62% of the HBM roofline).
constexpr int kFinVec = 4;
template <typename OutT, typename Idx>
__global__ void __launch_bounds__(256)
    finalize_kernel(Idx nunits, int BH, int H, int d4_shift, const float* __restrict__ acc_o,
                    const float* __restrict__ acc_lse, OutT* __restrict__ out, int64_t sB,
                    int64_t sH, int64_t sN, int64_t out_row0, int64_t n_total,
                    float* __restrict__ lse_out) {
  const Idx D4 = Idx(1) << d4_shift;
  const Idx n4 = nunits << d4_shift;
  const Idx stride = Idx(gridDim.x) * blockDim.x;
  for (Idx b = Idx(blockIdx.x) * blockDim.x + threadIdx.x; b < n4; b += stride * kFinVec) {
    float4 v[kFinVec];
    float l[kFinVec];
#pragma unroll
    for (int u = 0; u < kFinVec; ++u) {
      const Idx f = b + u * stride;
      if (f < n4) {
        v[u] = reinterpret_cast<const float4*>(acc_o)[f];
        l[u] = acc_lse ? acc_lse[f >> d4_shift] : 0.f;   // NULL: plain cast (backward)
      }
    }
#pragma unroll
    for (int u = 0; u < kFinVec; ++u) {
      const Idx f = b + u * stride;
      if (f >= n4) continue;
      const Idx unit = f >> d4_shift;
      const int d = int(f & (D4 - 1)) * 4;
      if (l[u] == -INFINITY) v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      const Idx r = unit / Idx(BH);
      const int p = int(unit - r * Idx(BH));
      const int bb = p / H, hh = p - bb * H;
      store4(out + int64_t(bb) * sB + int64_t(hh) * sH + (out_row0 + int64_t(r)) * sN + d, v[u]);
      if (d == 0 && lse_out) lse_out[int64_t(p) * n_total + out_row0 + int64_t(r)] = l[u];
    }
  }
}

cudaError_t launch_fill(float* p, int64_t n, float val, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  fill_f32_kernel<<<unsigned(blocks), 256, 0, st>>>(p, n, val);
  return cudaGetLastError();
}

cudaError_t launch_merge(int64_t rows, int B, int H, int D, int n_parts, const float* const* po,
                         const float* const* pl, float* acc_o, float* acc_lse, bool acc_write,
                         void* out, cqs_dtype out_dtype, const int64_t* out_strides,
                         int64_t out_row0, int64_t n_total, float* lse_out, cudaStream_t st) {
  MergeParts mp{};
  mp.n = n_parts;
  for (int j = 0; j < n_parts; ++j) {
    mp.o[j] = po[j];
    mp.l[j] = pl[j];
  }
  const int BH = B * H;
  const int64_t nunits = rows * BH;
  if (nunits <= 0) return cudaSuccess;
  const int64_t sB = out ? out_strides[0] : 0, sH = out ? out_strides[1] : 0,
                sN = out ? out_strides[2] : 0;
  const bool bf = out && out_dtype == CQS_BF16;
  if (n_parts == 0 && acc_o && !acc_write && out && (D & (D - 1)) == 0) {
    int shift = 0;
    while ((4 << shift) < D) ++shift;
    const int64_t n4 = nunits * (D / 4);
    const int64_t blocks = std::min<int64_t>((n4 + 256 * kFinVec - 1) / (256 * kFinVec), 148 * 32);
    const bool small = n4 + int64_t(blocks) * 256 * kFinVec < (int64_t(1) << 31);
#define CQS_FIN(T, I)                                                                           \
  finalize_kernel<T, I><<<unsigned(blocks), 256, 0, st>>>(                                      \
      I(nunits), BH, H, shift, acc_o, acc_lse, static_cast<T*>(out), sB, sH, sN, out_row0,      \
      n_total, lse_out)
    if (bf && small) CQS_FIN(__nv_bfloat16, uint32_t);
    else if (bf) CQS_FIN(__nv_bfloat16, int64_t);
    else if (small) CQS_FIN(float, uint32_t);
    else CQS_FIN(float, int64_t);
#undef CQS_FIN
    return cudaGetLastError();
  }
  const int D4 = D / 4, lpu = D4 < 32 ? D4 : 32, upw = 32 / lpu;
  const int64_t warps = (nunits + upw - 1) / upw;
  const int64_t blocks = std::min<int64_t>((warps + 7) / 8, 148 * 64);
  const bool small = nunits + int64_t(blocks) * 256 < (int64_t(1) << 31);
#define CQS_MERGE(T, NPV, I)                                                                   \
  merge_kernel<T, NPV, I><<<unsigned(blocks), 256, 0, st>>>(                                   \
      I(nunits), BH, H, D4, mp, acc_o, acc_lse, acc_write, static_cast<T*>(out), sB, sH, sN,   \
      out_row0, n_total, lse_out)
#define CQS_MERGE_NP(T, I)                          \
  if (n_parts <= 1) CQS_MERGE(T, 1, I);             \
  else if (n_parts <= 2) CQS_MERGE(T, 2, I);        \
  else if (n_parts <= 4) CQS_MERGE(T, 4, I);        \
  else if (n_parts <= 8) CQS_MERGE(T, 8, I);        \
  else CQS_MERGE(T, 16, I);
  if (bf) {
    if (small) { CQS_MERGE_NP(__nv_bfloat16, uint32_t) } else { CQS_MERGE_NP(__nv_bfloat16, int64_t) }
  } else {
    if (small) { CQS_MERGE_NP(float, uint32_t) } else { CQS_MERGE_NP(float, int64_t) }
  }
#undef CQS_MERGE_NP
#undef CQS_MERGE
  return cudaGetLastError();
}

}  // namespace cqs

extern "C" cqs_status cqs_merge(int64_t rows, int32_t B, int32_t H, int32_t D, int32_t n_parts,
                                const float* const* part_o, const float* const* part_lse,
                                float* acc_o, float* acc_lse, void* out, cqs_dtype out_dtype,
                                const int64_t out_strides[4], int64_t out_row0, int64_t n_total,
                                float* lse_out, void* stream) {
  using namespace cqs;
  if (rows < 0 || B < 1 || H < 1 || D < 4 || D > 256 || D % 4 != 0 || n_parts < 0 ||
      n_parts > kMaxMergeParts)
    return fail(CQS_E_INVALID, "cqs_merge: bad sizes (D % 4 == 0, D <= 256, n_parts <= 16)");
  if (n_parts > 0 && (!part_o || !part_lse)) return fail(CQS_E_INVALID, "cqs_merge: NULL parts");
  for (int j = 0; j < n_parts; ++j)
    if (!part_o[j] || !part_lse[j]) return fail(CQS_E_INVALID, "cqs_merge: NULL part pointer");
  if ((acc_o == nullptr) != (acc_lse == nullptr))
    return fail(CQS_E_INVALID, "cqs_merge: acc_o and acc_lse must both be set or both NULL");
  if (out && (!out_strides || out_strides[3] != 1))
    return fail(CQS_E_INVALID, "cqs_merge: out needs strides with stride(D) == 1");
  if ((out || lse_out) && (out_row0 < 0 || out_row0 + rows > n_total))
    return fail(CQS_E_INVALID, "cqs_merge: out rows out of range");
  const bool acc_write = acc_o && n_parts > 0;
  cudaError_t e = launch_merge(rows, B, H, D, n_parts, part_o, part_lse, acc_o, acc_lse, acc_write,
                               out, out_dtype, out_strides, out_row0, n_total, lse_out,
                               static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("cqs_merge: ") + cudaGetErrorString(e));
  return CQS_OK;
}

// ---------------------------------------------------------------------------------------------
// R-way SUM of fp32 partial gradients (multi-GPU backward, Alg. 2's IndexAdd across ranks,
// P:122-124): out[b,h,row0+r,:] = cast(sum_j part_j[r][p][:]).  Thread -> (unit, float4 column),
// all R loads in flight before the adds; parts may be peer (NVLink) pointers.
// ---------------------------------------------------------------------------------------------
namespace cqs {

template <typename OutT>
__global__ void __launch_bounds__(256)
    reduce_sum_kernel(int64_t nunits, int BH, int H, int d4_shift, MergeParts parts,
                      OutT* __restrict__ out, int64_t sB, int64_t sH, int64_t sN,
                      int64_t out_row0) {
  const int64_t n4 = nunits << d4_shift;
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < n4;
       f += int64_t(gridDim.x) * blockDim.x) {
    float4 v[kMaxMergeParts];
#pragma unroll
    for (int j = 0; j < kMaxMergeParts; ++j)
      if (j < parts.n) v[j] = reinterpret_cast<const float4*>(parts.o[j])[f];
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kMaxMergeParts; ++j)
      if (j < parts.n) s.x += v[j].x, s.y += v[j].y, s.z += v[j].z, s.w += v[j].w;
    const int64_t unit = f >> d4_shift;
    const int d = int(f & ((int64_t(1) << d4_shift) - 1)) * 4;
    const int64_t r = unit / BH;
    const int p = int(unit - r * BH);
    const int bb = p / H, hh = p - bb * H;
    store4(out + int64_t(bb) * sB + int64_t(hh) * sH + (out_row0 + r) * sN + d, s);
  }
}

}  // namespace cqs

extern "C" cqs_status cqs_reduce_sum(int64_t rows, int32_t B, int32_t H, int32_t D,
                                     int32_t n_parts, const float* const* parts, void* out,
                                     cqs_dtype out_dtype, const int64_t out_strides[4],
                                     int64_t out_row0, void* stream) {
  using namespace cqs;
  if (rows < 0 || B < 1 || H < 1 || D < 4 || D > 256 || (D & (D - 1)) != 0 || n_parts < 1 ||
      n_parts > kMaxMergeParts)
    return fail(CQS_E_INVALID, "cqs_reduce_sum: bad sizes (D a power of two in [4,256], 1..16 parts)");
  if (!parts || !out || !out_strides || out_strides[3] != 1 || out_row0 < 0)
    return fail(CQS_E_INVALID, "cqs_reduce_sum: NULL parts/out or stride(D) != 1");
  MergeParts mp{};
  mp.n = n_parts;
  for (int j = 0; j < n_parts; ++j) {
    if (!parts[j] || (reinterpret_cast<uintptr_t>(parts[j]) & 15))
      return fail(CQS_E_INVALID, "cqs_reduce_sum: NULL or non-16-byte-aligned part");
    mp.o[j] = parts[j];
  }
  const int64_t nunits = rows * int64_t(B) * H;
  if (nunits == 0) return CQS_OK;
  int shift = 0;
  while ((4 << shift) < D) ++shift;
  const int64_t n4 = nunits * (D / 4);
  const int64_t blocks = std::min<int64_t>((n4 + 255) / 256, 148 * 32);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (out_dtype == CQS_BF16)
    reduce_sum_kernel<__nv_bfloat16><<<unsigned(blocks), 256, 0, st>>>(
        nunits, B * H, H, shift, mp, static_cast<__nv_bfloat16*>(out), out_strides[0],
        out_strides[1], out_strides[2], out_row0);
  else
    reduce_sum_kernel<float><<<unsigned(blocks), 256, 0, st>>>(
        nunits, B * H, H, shift, mp, static_cast<float*>(out), out_strides[0], out_strides[1],
        out_strides[2], out_row0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("cqs_reduce_sum: ") + cudaGetErrorString(e));
  return CQS_OK;
}

// LSE merge / finalize kernels (Eq. 3 in LSE form, PAPER.md P:48-52 with Den_j = exp(lse_j),
// Num_j = O_j Den_j).  HBM-bound: one warp per (row, plane), 16-byte vector loads of the
// D-contiguous fp32 rows, coalesced across the warp; bf16/fp32 output cast fused.
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

// rows x planes, one warp each.  Parts are [rows][BH][D]; acc (optional) likewise.
template <typename OutT>
__global__ void __launch_bounds__(256)
    merge_kernel(int64_t rows, int BH, int H, int D, MergeParts parts, float* __restrict__ acc_o,
                 float* __restrict__ acc_lse, bool acc_write, OutT* __restrict__ out, int64_t sB,
                 int64_t sH, int64_t sN, int64_t out_row0, int64_t n_total,
                 float* __restrict__ lse_out) {
  const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= rows * BH) return;
  const int64_t r = wid / BH;
  const int p = int(wid % BH);
  const int64_t row_off = wid * D;
  // weights
  float mx = -INFINITY;
  const float la = acc_lse ? acc_lse[wid] : -INFINITY;
  mx = fmaxf(mx, la);
  for (int j = 0; j < parts.n; ++j) mx = fmaxf(mx, parts.l[j][wid]);
  float lse, wa = 0.f;
  float w[kMaxMergeParts];
  if (mx == -INFINITY) {
    lse = -INFINITY;
    for (int j = 0; j < kMaxMergeParts; ++j) w[j] = 0.f;
  } else {
    float s = 0.f;
    if (la != -INFINITY) {
      wa = expf(la - mx);
      s += wa;
    }
#pragma unroll
    for (int j = 0; j < kMaxMergeParts; ++j) {
      w[j] = 0.f;
      if (j < parts.n) {
        const float lj = parts.l[j][wid];
        if (lj != -INFINITY) w[j] = expf(lj - mx);
        s += w[j];
      }
    }
    const float inv = 1.f / s;
    wa *= inv;
#pragma unroll
    for (int j = 0; j < kMaxMergeParts; ++j) w[j] *= inv;
    lse = mx + logf(s);
  }
  OutT* orow = out ? out + int64_t(p / H) * sB + int64_t(p % H) * sH + (out_row0 + r) * sN : nullptr;
  for (int d = lane * 4; d < D; d += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (wa != 0.f) {
      const float4 a = *reinterpret_cast<const float4*>(acc_o + row_off + d);
      acc.x = wa * a.x, acc.y = wa * a.y, acc.z = wa * a.z, acc.w = wa * a.w;
    }
    for (int j = 0; j < parts.n; ++j) {
      if (w[j] == 0.f) continue;
      const float4 b = *reinterpret_cast<const float4*>(parts.o[j] + row_off + d);
      acc.x = fmaf(w[j], b.x, acc.x);
      acc.y = fmaf(w[j], b.y, acc.y);
      acc.z = fmaf(w[j], b.z, acc.z);
      acc.w = fmaf(w[j], b.w, acc.w);
    }
    if (acc_write) store4(acc_o + row_off + d, acc);
    if (orow) store4(orow + d, acc);
  }
  if (lane == 0) {
    if (acc_write) acc_lse[wid] = lse;
    if (lse_out) lse_out[int64_t(p) * n_total + out_row0 + r] = lse;
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
  const int64_t warps = rows * BH;
  if (warps <= 0) return cudaSuccess;
  const int64_t blocks = (warps * 32 + 255) / 256;
  const int64_t sB = out ? out_strides[0] : 0, sH = out ? out_strides[1] : 0,
                sN = out ? out_strides[2] : 0;
  if (!out || out_dtype == CQS_F32)
    merge_kernel<float><<<unsigned(blocks), 256, 0, st>>>(
        rows, BH, H, D, mp, acc_o, acc_lse, acc_write, static_cast<float*>(out), sB, sH, sN,
        out_row0, n_total, lse_out);
  else
    merge_kernel<__nv_bfloat16><<<unsigned(blocks), 256, 0, st>>>(
        rows, BH, H, D, mp, acc_o, acc_lse, acc_write, static_cast<__nv_bfloat16*>(out), sB, sH,
        sN, out_row0, n_total, lse_out);
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

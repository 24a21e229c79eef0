"""Seeded synthetic Q/K/V generator shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no chunking, no masks, no softmax): it only
turns (seed, tensor id, flat element index) into a number.  It is the single place both sides of
every parity test draw their inputs from.

Recipe (SURVEY.md §8d "Synthetic inputs"):
  h_j   = splitmix64_finalize(K0 * (4*seed + tid) + K1 * (3*e + j))   for j = 0, 1, 2   (mod 2^64)
  u_0..u_11 = the four 16-bit lanes of h_0, h_1, h_2
  x     = (sum_i u_i - 6 * 2^16) / 2^16          (Irwin-Hall(12): mean ~0, variance ~1, |x| <= 6)
where e is the row-major flat index over [B, H, N, D] and tid is 0 for Q, 1 for K, 2 for V, 3 for dO.
The integer sum is exact in fp32; bf16 inputs are the fp32 value rounded to nearest-even.

Two implementations with bit-identical results: `numpy_*` (uint64, well defined wrap-around) and
`torch_*` (int64 two's-complement wrap, runs on CPU or CUDA).  tests/test_synth.py checks they agree.
"""
from __future__ import annotations

import numpy as np

K0 = 0x9E3779B97F4A7C15
K1 = 0xD1B54A32D192ED03
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
TID = {"q": 0, "k": 1, "v": 2, "do": 3}   # "do": the upstream gradient dO of the backward
BASE_SEED = 20260417  # seed = 20260417 + config index


def _u64(x: int) -> np.uint64:
    return np.uint64(x & 0xFFFFFFFFFFFFFFFF)


def _np_mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _u64(M1)
    z = (z ^ (z >> np.uint64(27))) * _u64(M2)
    return z ^ (z >> np.uint64(31))


def numpy_values(seed: int, tid: int, start: int, count: int) -> np.ndarray:
    """fp32 values for flat indices [start, start+count) of tensor `tid`."""
    with np.errstate(over="ignore"):
        e = np.arange(start, start + count, dtype=np.uint64)
        base = _u64(K0 * (4 * seed + tid))
        tot = np.zeros(count, dtype=np.int64)
        for j in range(3):
            h = _np_mix(base + _u64(K1) * (np.uint64(3) * e + np.uint64(j)))
            for s in (0, 16, 32, 48):
                tot += ((h >> np.uint64(s)) & np.uint64(0xFFFF)).astype(np.int64)
    return ((tot - 6 * 65536).astype(np.float32)) / np.float32(65536.0)


def numpy_tensor(shape, seed: int, name: str, bf16: bool = False) -> np.ndarray:
    """Full tensor as float64 numpy array (values exactly representable in fp32 / bf16)."""
    n = int(np.prod(shape))
    x = numpy_values(seed, TID[name], 0, n)
    if bf16:
        x = round_bf16(x)
    return x.astype(np.float64).reshape(shape)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 round-to-nearest-even, returned as fp32 holding the bf16 value."""
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = (b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


# ---------------------------------------------------------------------------------------------
# torch implementation (same integers, int64 wrap-around); used to build large inputs on the GPU
# ---------------------------------------------------------------------------------------------

def _s64(x: int) -> int:
    x &= 0xFFFFFFFFFFFFFFFF
    return x - (1 << 64) if x >= (1 << 63) else x


def _t_shr(z, s: int):
    return (z >> s) & ((1 << (64 - s)) - 1)


def _t_mix(z):
    z = (z ^ _t_shr(z, 30)) * _s64(M1)
    z = (z ^ _t_shr(z, 27)) * _s64(M2)
    return z ^ _t_shr(z, 31)


def torch_values(seed: int, tid: int, start: int, count: int, device="cpu"):
    import torch
    e = torch.arange(start, start + count, dtype=torch.int64, device=device)
    base = _s64(K0 * (4 * seed + tid))
    tot = torch.zeros(count, dtype=torch.int64, device=device)
    for j in range(3):
        h = _t_mix(base + (3 * e + j) * _s64(K1))
        for s in (0, 16, 32, 48):
            tot += _t_shr(h, s) & 0xFFFF if s else h & 0xFFFF
    return (tot - 6 * 65536).to(torch.float32) / 65536.0


def torch_tensor(shape, seed: int, name: str, dtype=None, device="cpu", chunk: int = 1 << 25):
    """Tensor of `shape` (row-major flat index) in `dtype` (torch.float32 or torch.bfloat16)."""
    import torch
    dtype = dtype or torch.float32
    n = 1
    for s in shape:
        n *= int(s)
    out = torch.empty(n, dtype=dtype, device=device)
    for st in range(0, n, chunk):
        c = min(chunk, n - st)
        out[st:st + c] = torch_values(seed, TID[name], st, c, device).to(dtype)
    return out.view(*shape)


def torch_qkv(B, H, N, D, seed, dtype=None, device="cpu"):
    return tuple(torch_tensor((B, H, N, D), seed, nm, dtype, device) for nm in ("q", "k", "v"))

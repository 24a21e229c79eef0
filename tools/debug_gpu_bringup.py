"""Scratch diagnostics for the first GPU bring-up (prints, does not assert)."""
import math
import sys

import numpy as np
import torch

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O


def run(N, H, D, depth, bf16, label, mod=None):
    dt = torch.bfloat16 if bf16 else torch.float32
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 1234, dtype=dt, device="cuda")
    if mod:
        q, k, v = mod(q, k, v)
    try:
        out, lse = cqs.attention(q, k, v, depth=depth)
        torch.cuda.synchronize()
    except Exception as e:
        print(label, "EXC", e)
        return
    Oref, lref = O.dense_attention(*(t.double().cpu().numpy() for t in (q, k, v)))
    o = out.double().cpu().numpy()
    print("%-28s maxerr %.3e  ref max %.3e  lse err %.3e  nan %d" % (
        label, np.nanmax(np.abs(o - Oref)), np.abs(Oref).max(),
        np.nanmax(np.abs(lse.double().cpu().numpy() - lref)), int(np.isnan(o).sum())))
    sys.stdout.flush()


if __name__ == "__main__":
    run(448, 1, 64, 1, False, "f32 C1")
    run(1030, 2, 64, 2, False, "f32 d2")
    # bf16 special inputs: K = 0 -> uniform P: tests PV path only
    z = lambda q, k, v: (q, torch.zeros_like(k), v)
    run(128, 1, 128, 0, True, "bf16 K=0 N=128 d0", z)
    run(256, 1, 128, 0, True, "bf16 K=0 N=256 d0", z)
    # V = const ones column pattern: tests QK + softmax
    def vconst(q, k, v):
        v2 = torch.zeros_like(v)
        v2[..., 0] = 1
        return q, k, v2
    run(128, 1, 128, 0, True, "bf16 V=e0 N=128 d0", vconst)
    run(128, 1, 128, 0, True, "bf16 N=128 d0")
    run(300, 1, 128, 0, True, "bf16 N=300 d0")
    run(1030, 2, 128, 1, True, "bf16 N=1030 d1")
    run(1030, 2, 64, 1, True, "bf16 D64 N=1030 d1")
    run(2401, 2, 128, 3, True, "bf16 N=2401 d3")

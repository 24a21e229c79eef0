"""Small invocations of every libcqs device path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck; tools/sanitize.sh).  Run with PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every
tensor is its own cudaMalloc and an out-of-bounds access cannot hide inside a cached block.
Checks the results against tools/_rowref.py so a silent corruption also fails the run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import cqs_synth  # noqa: E402
import paper_2604_20819_b200 as cqs  # noqa: E402
from tools import _rowref as R  # noqa: E402


def check(out, lse, q, k, v, tol):
    rows = np.array([0, q.shape[2] // 3, q.shape[2] - 1])
    for h in range(q.shape[1]):
        o, l_ = R.rows_forward(*(t[0, h].double().cpu().numpy() for t in (q, k, v)), rows)
        assert np.abs(out[0, h].double().cpu().numpy()[rows] - o).max() <= tol
        assert np.abs(lse[0, h].double().cpu().numpy()[rows] - l_).max() <= 1e-3


def main():
    which = sys.argv[1:] or ["c1", "bf16_128", "bf16_64", "streamed", "merge", "bwd"]
    dev = "cuda"
    if "c1" in which:      # BASELINE config 0: fp32, N=448, D=64, one level
        q, k, v = cqs_synth.torch_qkv(1, 1, 448, 64, 1, torch.float32, dev)
        out, lse = cqs.attention(q, k, v, depth=1)
        check(out, lse, q, k, v, 1e-5)
    if "bf16_128" in which:   # CTA-pair kernel: ragged tiles, depth 2, two heads
        q, k, v = cqs_synth.torch_qkv(1, 2, 1300, 128, 2, torch.bfloat16, dev)
        out, lse = cqs.attention(q, k, v, depth=2)
        check(out, lse, q, k, v, 2e-2)
    if "bf16_64" in which:
        q, k, v = cqs_synth.torch_qkv(1, 2, 1300, 64, 3, torch.bfloat16, dev)
        out, lse = cqs.attention(q, k, v, depth=2)
        check(out, lse, q, k, v, 2e-2)
    if "streamed" in which:   # pinned-host Q/K/V, host-tier accumulator, one staging buffer
        q, k, v = (t.pin_memory() for t in cqs_synth.torch_qkv(1, 2, 2000, 128, 4, torch.bfloat16))
        d = cqs.make_desc(N=2000, B=1, H=2, D=128, depth=2, in_dtype="bf16", qkv_loc="host")
        budget, _ = cqs.cqs_memory_model(d, 2, 1, 1)
        p = cqs.cqs_plan(N=2000, B=1, H=2, D=128, depth=2, budget_bytes=budget, in_dtype="bf16",
                         qkv_loc="host", out_loc="host")
        dv, hb = cqs.cqs_forward_workspace_size(p)
        ws = torch.empty(dv, dtype=torch.uint8, device=dev)
        hws = torch.empty(max(hb, 256), dtype=torch.uint8).pin_memory() if hb else None
        out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
        lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()
        cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, budget, ws, hws)
        torch.cuda.synchronize()
        check(out, lse, q, k, v, 2e-2)
    if "merge" in which:
        rows, B, H, D = 777, 1, 3, 128
        po = [torch.randn(rows, B * H, D, device=dev) for _ in range(4)]
        pl = [torch.randn(rows, B * H, device=dev) for _ in range(4)]
        out = torch.empty(B, H, rows, D, device=dev)
        lse = torch.empty(B, H, rows, device=dev)
        cqs.cqs_merge(rows, B, H, D, po, pl, out=out, lse_out=lse)
        torch.cuda.synchronize()
    if "bwd" in which:
        q, k, v = cqs_synth.torch_qkv(1, 2, 1100, 128, 5, torch.bfloat16, dev)
        do = cqs_synth.torch_tensor((1, 2, 1100, 128), 5, "do", torch.bfloat16, dev)
        out, lse = cqs.attention(q, k, v, depth=2)
        g = cqs.attention_backward(q, k, v, out, do, lse, depth=2, grad_dtype=torch.float32)
        torch.cuda.synchronize()
        assert all(torch.isfinite(x).all() for x in g)
    torch.cuda.synchronize()
    print("sanitize cases ok:", " ".join(which))


if __name__ == "__main__":
    main()

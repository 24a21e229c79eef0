"""Backward (Algorithm 2) throughput on the C2 shape: N=131072, H=32, D=128 (or --D 64), bf16,
depth 1, resident.  Algorithmic FLOPs per step = 10 N^2 D B H (S, dP, dV, dK, dQ: five N x N x D
products; the kernels execute 14 N^2 D because dQ runs in its own kernel and recomputes S and dP).

    python tools/bwd_bench.py [--D 128] [--steps 5] [--warmup 3] > profiles/rNN_bwd.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=131072)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    B, H, N, D = 1, a.H, a.N, a.D
    q, k, v = cqs_synth.torch_qkv(B, H, N, D, 20260418, dtype=torch.bfloat16, device="cuda")
    do = cqs_synth.torch_tensor((B, H, N, D), 20260418, "do", torch.bfloat16, "cuda")
    out, lse = cqs.attention(q, k, v, depth=a.depth)
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=a.depth, in_dtype="bf16")
    ws = torch.empty(cqs.cqs_backward_workspace_size(p), dtype=torch.uint8, device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    for _ in range(a.warmup):
        cqs.cqs_attention_backward(p, q, k, v, out, do, lse, dq, dk, dv, 0.0, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        cqs.cqs_attention_backward(p, q, k, v, out, do, lse, dq, dk, dv, 0.0, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    st = cqs.cqs_attention_backward(p, q, k, v, out, do, lse, dq, dk, dv, 0.0, ws, stats=True)
    flops = 10.0 * N * N * D * B * H
    print(json.dumps({
        "what": "CQS backward (Algorithm 2), tcgen05 dK/dV + dQ kernels per task",
        "N": N, "H": H, "D": D, "depth": a.depth, "ms_per_step": ms,
        "tflops_algorithmic": flops / (ms * 1e-3) / 1e12,
        "tflops_executed": 1.4 * flops / (ms * 1e-3) / 1e12,
        "ms_task_kernels": st.ms_attn, "ms_prep_cast": st.ms_merge,
        "kernel_tflops_algorithmic": flops / (st.ms_attn * 1e-3) / 1e12,
        "launches": st.kernel_launches, "workspace_bytes": ws.numel()}))


if __name__ == "__main__":
    main()

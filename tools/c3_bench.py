"""BASELINE config 2: N = 1,000,000 tokens, 32 heads, D = 128, bf16, Q/K/V (and O, lse) in pinned
host memory, 16 GiB device budget -> the planner picks two CQS levels (49 tasks).  Times one full
streamed forward through the public C ABI and reports throughput, peak device memory against the
budget, H2D traffic and sampled-row parity against an fp64 sampled-row reference (tools/_rowref.py).

    python tools/c3_bench.py > profiles/r01_c3_streamed.json
    python tools/c3_bench.py --N 16777216 --H 1 --D 64 --budget-gib 1 --runs 1   # deep tree (NEXT-4)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from tools import _rowref as R

    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1_000_000)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--runs", type=int, default=2)
    args = ap.parse_args()
    B, H, N, D = 1, args.H, args.N, args.D
    budget = int(args.budget_gib * (1 << 30))
    seed = 20260419
    q, k, v = (cqs_synth.torch_tensor((B, H, N, D), seed, nm, torch.bfloat16, "cuda").cpu()
               .pin_memory() for nm in ("q", "k", "v"))
    torch.cuda.empty_cache()
    plan = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=-1, budget_bytes=budget, in_dtype="bf16",
                        qkv_loc="host", out_loc="host")
    info = plan.info()
    dev, host = cqs.cqs_forward_workspace_size(plan)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    ws = torch.empty(max(dev, 256), dtype=torch.uint8, device="cuda")
    hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
    out = torch.empty((B, H, N, D), dtype=torch.bfloat16).pin_memory()
    lse = torch.empty((B, H, N), dtype=torch.float32).pin_memory()
    cqs.attention(*(t[:, :min(2, H), :8192].cuda() for t in (q, k, v)), depth=1)   # warm-up
    torch.cuda.synchronize()
    res = {"config": "%sN=%d, H=%d, D=%d, bf16, QKV/O in pinned host memory, %.4g GiB budget" % (
               "C3: " if (N, H, D, args.budget_gib) == (1_000_000, 32, 128, 16.0) else "", N, H, D,
               args.budget_gib),
           "depth": info.depth, "tasks": info.n_tasks, "acc_depth": info.acc_depth,
           "stage_buffers": info.n_stage_buffers, "budget_bytes": budget,
           "predicted_peak_bytes": info.predicted_peak_bytes, "runs": []}
    for _ in range(args.runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = cqs.cqs_attention_forward(plan, q, k, v, out, lse, 0.0, budget, ws, hws, stats=True)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        res["runs"].append({"seconds": s, "tflops": 4.0 * N * N * D * H / s / 1e12,
                            "tokens_per_s": N / s, "bytes_h2d": st.bytes_h2d,
                            "bytes_d2h": st.bytes_d2h, "kernel_launches": st.kernel_launches})
    res["measured_peak_dev_bytes"] = torch.cuda.max_memory_allocated() - base
    # host link reference: best-of-5 pinned 1 GiB H2D / D2H
    hb = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    db = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: db.copy_(hb, non_blocking=True)),
                     ("d2h", lambda: hb.copy_(db, non_blocking=True))):
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        res["pcie_%s_gbs" % name] = (1 << 30) / (best * 1e-3) / 1e9
    del hb, db
    res["peak_within_budget"] = res["measured_peak_dev_bytes"] <= budget + 512
    rng = np.random.default_rng(9)
    errs, lerrs = [], []
    for h in rng.choice(H, min(2, H), replace=False):
        rows = np.sort(rng.choice(N, 8, replace=False))
        Oref, lref = R.rows_forward(q[0, h].double().numpy(), k[0, h].double().numpy(),
                                            v[0, h].double().numpy(), rows, block=1 << 18)
        errs.append(float(np.abs(out[0, h, rows].double().numpy() - Oref).max()))
        lerrs.append(float(np.abs(lse[0, h, rows].double().numpy() - lref).max()))
    res["parity"] = {"rows": 16, "max_abs_err": max(errs), "max_lse_err": max(lerrs)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()

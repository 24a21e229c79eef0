"""BASELINE config 3 (C4: N = 2^24 tokens, D = 128, bf16, tasks sharded over 1/2/4/8 B200) on the
one GPU this round has: every rank's share of the world-R plan is run back to back on the same
device (each rank's forward = its LPT tasks into its fp32 partial accumulator, exactly what rank r
executes on an R-GPU box before the single exchange), timed with CUDA events.  Reports per-rank
seconds, the makespan (what an R-GPU run waits for), the balance mean/max, and the projected
R-GPU throughput = total FLOPs / makespan.  The exchange (one peer-memory merge per rank, ~30 GB
read over NVLink per rank at R = 8) is not included and not measured here.

H = 4 instead of 8: heads are independent planes and the 8-head resident problem (QKV 103 GB +
69 GB accumulator) leaves no headroom on one 180 GB device; per-rank work scales linearly in H.

    python tools/c4_shards.py [--worlds 8 4 2] [--H 4] > profiles/r01_c4_shards.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1 << 24)
    ap.add_argument("--H", type=int, default=4)
    ap.add_argument("--worlds", type=int, nargs="+", default=[8, 4, 2])
    ap.add_argument("--schedule", default="hybrid")
    a = ap.parse_args()
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    N, H, D = a.N, a.H, 128
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 20260420, dtype=torch.bfloat16, device="cuda")
    flops = 4.0 * N * N * D * H
    res = {"config": "C4 shards: N=%d, H=%d, D=128, bf16, resident, %s schedule, base depth 1"
                     % (N, H, a.schedule), "total_tflop": flops / 1e12, "worlds": {}}
    ws = None
    for R in a.worlds:
        per = []
        for r in range(R):
            p = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=1, in_dtype="bf16", world=R, rank=r,
                             schedule=a.schedule)
            info = p.info()
            need, _ = cqs.cqs_forward_workspace_size(p)
            if ws is None or ws.numel() < need:
                ws = None
                torch.cuda.empty_cache()
                ws = torch.empty(need, dtype=torch.uint8, device="cuda")
            if R == a.worlds[0] and r == 0:   # warm once (kernel attributes, descriptors)
                cqs.attention(q[:, :, :8192], k[:, :, :8192], v[:, :, :8192], depth=1)
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cqs.cqs_attention_forward(p, q, k, v, None, None, 0.0, 0, ws, None)
            e1.record()
            torch.cuda.synchronize()
            s = e0.elapsed_time(e1) / 1e3
            per.append({"rank": r, "seconds": s, "tasks": info.my_tasks,
                        "work_frac": info.my_work_pairs / info.total_work_pairs,
                        "tflops": flops * info.my_work_pairs / info.total_work_pairs / s / 1e12})
            print(json.dumps({"R": R, **per[-1]}), file=sys.stderr, flush=True)
        mk = max(x["seconds"] for x in per)
        tot = sum(x["seconds"] for x in per)
        res["worlds"][str(R)] = {
            "tasks": info.n_tasks, "max_depth": info.max_depth, "per_rank": per,
            "makespan_s": mk, "sum_s": tot, "balance_mean_over_max": tot / R / mk,
            "projected_tflops_R_gpus": flops / mk / 1e12,
            "projected_efficiency_vs_1gpu_sum": tot / (R * mk)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()

"""BASELINE config 3 (C4: N = 2^24 tokens, D = 128, bf16, tasks sharded over 1/2/4/8 B200) on the
one GPU this round has: every rank's share of the world-R plan is run back to back on the same
device (each rank's forward = its LPT tasks into its fp32 partial accumulator, exactly what rank r
executes on an R-GPU box before the single exchange), timed with CUDA events.  Reports per-rank
seconds, the makespan (what an R-GPU run waits for), the balance mean/max, and the projected
R-GPU throughput = total FLOPs / makespan (+ the exchange: the owner's R-way merge of its shard,
timed here on local buffers of the real shard shape; over NVLink the peer reads add ~shard bytes /
link bandwidth, ~0.1% of the makespan).

Round 2: the full C4 config (H = 8, depth 3, contiguous DFS sharding): each rank's plan holds the
103 GB Q/K/V replica plus its rank-local accumulator (held rows only) — the layout an 8-GPU box
runs — so every rank's share is timed exactly as it would execute.

    python tools/c4_shards.py [--worlds 8 4] [--H 8] [--depth 3] [--shard contiguous]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1 << 24)
    ap.add_argument("--H", type=int, default=8)
    ap.add_argument("--worlds", type=int, nargs="+", default=[8, 4])
    ap.add_argument("--schedule", default="uniform")
    ap.add_argument("--shard", default="contiguous")
    ap.add_argument("--depth", type=int, default=3)
    a = ap.parse_args()
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    N, H, D = a.N, a.H, 128
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 20260420, dtype=torch.bfloat16, device="cuda")
    flops = 4.0 * N * N * D * H
    res = {"config": "C4 shards: N=%d, H=%d, D=128, bf16, resident replica + rank-local "
                     "accumulator, %s schedule, %s sharding, depth %d"
                     % (N, H, a.schedule, a.shard, a.depth), "total_tflop": flops / 1e12,
           "worlds": {}}
    ws = None
    for R in a.worlds:
        per = []
        for r in range(R):
            p = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=a.depth, in_dtype="bf16", world=R,
                             rank=r, schedule=a.schedule, shard=a.shard)
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
                        "predicted_peak_bytes": info.predicted_peak_bytes,
                        "acc_rows_frac": info.acc_rows / N,
                        "work_frac": info.my_work_pairs / info.total_work_pairs,
                        "tflops": flops * info.my_work_pairs / info.total_work_pairs / s / 1e12})
            print(json.dumps({"R": R, **per[-1]}), file=sys.stderr, flush=True)
        mk = max(x["seconds"] for x in per)
        tot = sum(x["seconds"] for x in per)
        # the exchange: R-way merge of one shard (rows N/R, fp32 partials -> bf16 O + lse), timed
        # on local buffers (the workspace is released first: the shard parts are small)
        ws = None
        torch.cuda.empty_cache()
        rows = N // R
        parts_o = [torch.randn(rows, H, D, device="cuda") for _ in range(R)]
        parts_l = [torch.randn(rows, H, device="cuda") for _ in range(R)]
        out = torch.empty(1, H, rows, D, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(1, H, rows, device="cuda")
        cqs.cqs_merge(rows, 1, H, D, parts_o, parts_l, out=out, lse_out=lse)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cqs.cqs_merge(rows, 1, H, D, parts_o, parts_l, out=out, lse_out=lse)
        e1.record()
        torch.cuda.synchronize()
        merge_s = e0.elapsed_time(e1) / 1e3
        del parts_o, parts_l, out, lse
        torch.cuda.empty_cache()
        res["worlds"][str(R)] = {
            "tasks": info.n_tasks, "max_depth": info.max_depth, "per_rank": per,
            "makespan_s": mk, "sum_s": tot, "balance_mean_over_max": tot / R / mk,
            "exchange_merge_s": merge_s,
            "projected_tflops_R_gpus": flops / (mk + merge_s) / 1e12,
            "projected_efficiency_vs_1gpu_sum": tot / (R * mk)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()

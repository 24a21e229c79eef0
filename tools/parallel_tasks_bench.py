"""Tasks in flight (n_parallel) on trees whose single tasks do not fill the GPU: time
cqs_attention_forward at n_parallel = 1, 2, 4, 8 (resident, CUDA events, best of 3).

    python tools/parallel_tasks_bench.py [--N 120000] [--H 1] [--D 64] [--depth 6]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=120000)
    ap.add_argument("--H", type=int, default=1)
    ap.add_argument("--D", type=int, default=64)
    ap.add_argument("--depth", type=int, default=6)
    a = ap.parse_args()
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    q, k, v = cqs_synth.torch_qkv(1, a.H, a.N, a.D, 5, torch.bfloat16, "cuda")
    out = torch.empty_like(q)
    lse = torch.empty(1, a.H, a.N, dtype=torch.float32, device="cuda")
    flops = 4.0 * a.N * a.N * a.D * a.H
    res = {"config": "N=%d H=%d D=%d depth %d (resident)" % (a.N, a.H, a.D, a.depth), "runs": []}
    for P in (1, 2, 4, 8):
        p = cqs.cqs_plan(N=a.N, B=1, H=a.H, D=a.D, depth=a.depth, n_parallel=P)
        ws = torch.empty(cqs.cqs_forward_workspace_size(p)[0], dtype=torch.uint8, device="cuda")
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, None)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res["runs"].append({"n_parallel": P, "ms": best, "tflops": flops / (best * 1e-3) / 1e12,
                            "tasks": p.info().my_tasks})
        print(json.dumps(res["runs"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

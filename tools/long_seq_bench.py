"""Forward throughput on long single-head sequences (the C5 regime: every work item loops over
thousands of KV tiles, so the CTAs in flight stay in lock step for the whole task), resident.

    python tools/long_seq_bench.py [--N 4194304] [--D 64] [--H 1] [--depth 1] [--runs 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4194304)
    ap.add_argument("--D", type=int, default=64)
    ap.add_argument("--H", type=int, default=1)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--runs", type=int, default=2)
    a = ap.parse_args()
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    q, k, v = cqs_synth.torch_qkv(1, a.H, a.N, a.D, 20260421, dtype=torch.bfloat16, device="cuda")
    cqs.attention(q[:, :, :8192], k[:, :, :8192], v[:, :, :8192], depth=1)
    torch.cuda.synchronize()
    res = []
    for _ in range(a.runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cqs.attention(q, k, v, depth=a.depth)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        res.append({"seconds": s, "tflops": 4.0 * a.N * a.N * a.D * a.H / s / 1e12})
    print(json.dumps({"N": a.N, "H": a.H, "D": a.D, "depth": a.depth, "runs": res,
                      "lib": os.path.basename(cqs.LIB_PATH)}))


if __name__ == "__main__":
    main()

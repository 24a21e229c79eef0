"""R-way LSE merge (cqs_merge, Eq. 3) at the multi-GPU exchange's shape: the owner of one
row shard of C4 (N = 2^24, H = 8, D = 128, R = 8 ranks -> 2^21 rows) merges R partials and writes
the bf16 O / fp32 lse shard.  Algorithmic bytes per launch: R x rows x B*H x (D+1) x 4 read +
rows x B*H x (D x 2 + 4) written.  Prints one JSON line (CUDA-event timing); run under ncu for the
dram counters:  python tools/merge_bench.py [--parts 8] [--rows 2097152]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--rows", type=int, default=1 << 21)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_2604_20819_b200 as cqs
    R, rows, B, H, D = args.parts, args.rows, 1, args.heads, 128
    po = [torch.randn(rows, B * H, D, device="cuda") for _ in range(R)]
    pl = [torch.randn(rows, B * H, device="cuda") for _ in range(R)]
    out = torch.empty(B, H, rows, D, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B, H, rows, device="cuda")
    for _ in range(2):
        cqs.cqs_merge(rows, B, H, D, po, pl, out=out, lse_out=lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        cqs.cqs_merge(rows, B, H, D, po, pl, out=out, lse_out=lse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    nbytes = R * rows * B * H * (D + 1) * 4 + rows * B * H * (D * 2 + 4)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = None
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": "merge_kernel<bf16> (cqs_merge)", "parts": R, "rows": rows,
                      "heads": H, "D": D, "ms_per_launch": ms, "algorithmic_bytes": nbytes,
                      "achieved_gbs": gbs, "peak_hbm_gbs": peak,
                      "frac": gbs / peak if peak else None}))


if __name__ == "__main__":
    main()

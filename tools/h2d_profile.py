"""Host-to-device copy rates of the streamed executor from CUDA activity records (CUPTI through
torch.profiler — the image has no nsys): every memcpy the library issues during one streamed
forward (per-task segment staging H2D, output / flush D2H) with its bytes and duration.
C2 shape by default (N = 131072, H = 32, D = 128, Q/K/V/O in pinned host memory).

    python tools/h2d_profile.py [--N 131072] [--H 32] [--depth 1] > profiles/r02_h2d_profile.json"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=131072)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--budget-gib", type=float, default=0.0)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    N, H, D = args.N, args.H, args.D
    q, k, v = (cqs_synth.torch_tensor((1, H, N, D), 20260418, nm, torch.bfloat16, "cuda").cpu()
               .pin_memory() for nm in ("q", "k", "v"))
    budget = int(args.budget_gib * (1 << 30))
    kw = dict(N=N, B=1, H=H, D=D, depth=args.depth if not budget else -1, budget_bytes=budget,
              in_dtype="bf16", qkv_loc="host", out_loc="host")
    p = cqs.cqs_plan(**kw)
    dv, hb = cqs.cqs_forward_workspace_size(p)
    ws = torch.empty(dv, dtype=torch.uint8, device="cuda")
    hws = torch.empty(max(hb, 256), dtype=torch.uint8).pin_memory() if hb else None
    out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
    lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()
    cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, hws)   # warm-up
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        st = cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, hws, stats=True)
        torch.cuda.synchronize()
    copies = {"HtoD": [0, 0.0, 0, float("inf"), 0.0], "DtoH": [0, 0.0, 0, float("inf"), 0.0]}
    kern_us, t_lo, t_hi = 0.0, float("inf"), 0.0
    for ev in prof.events():
        name = ev.name
        dur = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        t_lo = min(t_lo, ev.time_range.start)
        t_hi = max(t_hi, ev.time_range.end)
        if "Memcpy" in name:
            kind = "HtoD" if "HtoD" in name else ("DtoH" if "DtoH" in name else None)
            if kind is None:
                continue
            nbytes = getattr(ev, "bytes", 0) or 0
            c = copies[kind]
            c[0] += 1
            c[1] += ev.time_range.end - ev.time_range.start
            c[2] += nbytes
            c[3] = min(c[3], ev.time_range.start)
            c[4] = max(c[4], ev.time_range.end)
        elif "Memset" not in name:
            kern_us += dur
    res = {"config": "streamed forward N=%d H=%d D=%d depth %d" % (N, H, D, p.info().depth),
           "library_bytes_h2d": st.bytes_h2d, "library_bytes_d2h": st.bytes_d2h,
           "wall_ms_stats": st.ms_total}
    for kind, (n, busy_us, nbytes, lo, hi) in copies.items():
        nb = nbytes or (st.bytes_h2d if kind == "HtoD" else st.bytes_d2h)
        res[kind] = {"copies": n, "busy_ms": busy_us / 1e3, "span_ms": (hi - lo) / 1e3 if n else 0,
                     "bytes": nb, "bytes_source": "cupti" if nbytes else "library counters",
                     "gbs_while_busy": nb / (busy_us * 1e-6) / 1e9 if busy_us else None,
                     "gbs_over_span": nb / ((hi - lo) * 1e-6) / 1e9 if n else None}
    res["profiled_span_ms"] = (t_hi - t_lo) / 1e3
    print(json.dumps(res))


if __name__ == "__main__":
    main()

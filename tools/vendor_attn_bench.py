#!/usr/bin/env python
"""Same-box context for the attention kernels: library dense FMHA kernels on the C2 shape.

    python tools/vendor_attn_bench.py [--D 128 64] [--steps 5] [--warmup 3] [--out f.json]

Times, on the same GPU and in the same process, full (non-causal) softmax attention over
Q, K, V of shape [1, 32, 131072, D] bf16 (BASELINE configs[1]) through
  - cqs:       this repo's CQS path (cqs.attention, one CQS level, 7 tasks: bench.py's step)
  - cudnn:     torch SDPA with the cuDNN backend (NVIDIA's fused attention for sm_100)
  - torch_fa:  torch SDPA with its built-in flash backend
  - flash_attn: flash_attn.flash_attn_func (FA2, mma.sync, recompiled for sm_100)
Each: W warm-up calls, then K calls between CUDA events on the launch stream; inputs 1-3 GB >> L2.
TFLOP/s = 4 N^2 D H / time (every (q, k) pair once: the dense kernels and the CQS path do the same
useful work).  SM clocks / throttle reasons are sampled during each backend's timed region
(bench.ClockSampler), since all of these kernels run into the ~1 kW power cap.  A library that is
missing or refuses the shape is reported with the error, not skipped silently.  Measurement only:
nothing here is on the product path.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_calls(fn, args):
    import torch
    from bench import ClockSampler
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as cs:
        e0.record(st)
        for _ in range(args.steps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.steps, cs.summary()


def bwd_run(be, D, q, k, v, do, o_c, lse_c, flops, args):
    """Backward time of one backend: ours directly; library ones as (fwd + bwd) - fwd."""
    import torch
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel
    import paper_2604_20819_b200 as cqs
    row = {"backend": be, "D": D, "pass": "backward"}
    try:
        if be == "cqs":
            ms, clk = time_calls(lambda: cqs.attention_backward(q, k, v, o_c, do, lse_c, depth=1), args)
        else:
            if be == "cudnn":
                ctx = lambda: sdpa_kernel(SDPBackend.CUDNN_ATTENTION)
                f = lambda a, b, c: F.scaled_dot_product_attention(a, b, c)
            elif be == "torch_fa":
                ctx = lambda: sdpa_kernel(SDPBackend.FLASH_ATTENTION)
                f = lambda a, b, c: F.scaled_dot_product_attention(a, b, c)
            elif be == "flash_attn":
                from flash_attn import flash_attn_func
                import contextlib
                ctx = contextlib.nullcontext
                f = lambda a, b, c: flash_attn_func(a.transpose(1, 2), b.transpose(1, 2),
                                                    c.transpose(1, 2)).transpose(1, 2)
            else:
                raise ValueError(be)
            qg, kg, vg = (t.detach().clone().requires_grad_(True) for t in (q, k, v))

            def fb():
                with ctx():
                    o = f(qg, kg, vg)
                o.backward(do)
                qg.grad = kg.grad = vg.grad = None

            def fo():
                with ctx(), torch.no_grad():
                    f(qg, kg, vg)
            ms_fb, clk = time_calls(fb, args)
            ms_f, _ = time_calls(fo, args)
            ms = ms_fb - ms_f
            row["ms_fwd_plus_bwd"] = ms_fb
        row.update(ms=ms, tflops=flops / (ms * 1e-3) / 1e12, clocks=clk)
    except Exception as ex:
        row["error"] = ("%s: %s" % (type(ex).__name__, ex)).splitlines()[0][:300]
    torch.cuda.empty_cache()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", type=int, nargs="+", default=[128, 64])
    ap.add_argument("--N", type=int, default=131072)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--backends", nargs="+", default=["cqs", "cudnn", "torch_fa", "flash_attn"])
    ap.add_argument("--bwd", action="store_true",
                    help="time the backward instead (10 N^2 D H algorithmic FLOPs): ours = "
                         "cqs.attention_backward, cuDNN / FA = autograd of SDPA (fwd+bwd minus fwd)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel

    import cqs_synth
    from bench import ClockSampler
    import paper_2604_20819_b200 as cqs

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    res = {"gpu": torch.cuda.get_device_name(0), "N": args.N, "H": args.H, "steps": args.steps,
           "warmup": args.warmup, "cudnn": torch.backends.cudnn.version(), "runs": []}
    for D in args.D:
        q, k, v = cqs_synth.torch_qkv(1, args.H, args.N, D, 20260418, dtype=torch.bfloat16,
                                      device=dev)
        flops = (10.0 if args.bwd else 4.0) * args.N * args.N * D * args.H
        ref_out = None
        if args.bwd:
            do = cqs_synth.torch_tensor((1, args.H, args.N, D), 20260418, "do", torch.bfloat16, dev)
            o_c, lse_c = cqs.attention(q, k, v, depth=1)
        for be in args.backends:
            if args.bwd:
                res["runs"].append(bwd_run(be, D, q, k, v, do, o_c, lse_c, flops, args))
                print(json.dumps(res["runs"][-1]), flush=True)
                continue
            row = {"backend": be, "D": D}
            try:
                if be == "cqs":
                    fn = lambda: cqs.attention(q, k, v, depth=1)[0]
                elif be == "cudnn":
                    def fn():
                        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                            return F.scaled_dot_product_attention(q, k, v)
                elif be == "torch_fa":
                    def fn():
                        with sdpa_kernel(SDPBackend.FLASH_ATTENTION):
                            return F.scaled_dot_product_attention(q, k, v)
                elif be == "flash_attn":
                    from flash_attn import flash_attn_func
                    qt, kt, vt = (t.transpose(1, 2).contiguous() for t in (q, k, v))
                    fn = lambda: flash_attn_func(qt, kt, vt).transpose(1, 2)
                else:
                    raise ValueError(be)
                for _ in range(args.warmup):
                    o = fn()
                torch.cuda.synchronize()
                st = torch.cuda.current_stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with ClockSampler(0) as cs:
                    e0.record(st)
                    for _ in range(args.steps):
                        o = fn()
                    e1.record(st)
                    torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
                row.update(ms=ms, tflops=flops / (ms * 1e-3) / 1e12, clocks=cs.summary())
                # cross-check: every backend returns the same attention (sampled rows)
                o = o.float()
                if ref_out is None:
                    ref_out = o[0, :, ::4099].clone()
                row["max_abs_diff_vs_first"] = float((o[0, :, ::4099] - ref_out).abs().max())
                del o
            except Exception as ex:   # report, do not hide
                row["error"] = ("%s: %s" % (type(ex).__name__, ex)).splitlines()[0][:300]
            torch.cuda.empty_cache()
            print(json.dumps(row), flush=True)
            res["runs"].append(row)
        del q, k, v
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

"""BASELINE config 4 (N = 1e9 tokens, 1 head, D = 64, bf16, QKV in pinned host memory, one B200)
by the paper's own scaled evaluation (Sec. 3.3): one CQS Divide of
N' = 1e9 * (3/7)^(itr-1) tokens yields 7 leaves of the size the full itr-level tree has, streamed
from pinned host memory through the public C ABI (cqs_attention_forward, qkv_loc = out_loc =
pinned host).  Measured: t7 and the useful FLOP rate.  Extrapolated two ways:
  paper   : t_1B = t7 * 7^(itr-1)                         (Table 1 "Est. t_fwd")
  by work : t_1B = 4 N^2 D / (measured useful FLOP rate)  (at itr=6 ~40% of leaves are
            empty and kept area shrinks by (7/9)^itr, so counting leaves over-estimates)
Parity: sampled output rows against an fp64 sampled-row reference (tools/_rowref.py) over all N' keys.

    python tools/c5_scaled.py [--itr 6] [--rows 8] > profiles/r01_c5_scaled.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--itr", type=int, default=6)
    ap.add_argument("--rows", type=int, default=8)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--no-bwd", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from tools import _rowref as R

    N_full, H, D = 10 ** 9, 1, 64
    Np = int(round(N_full * (3 / 7) ** (args.itr - 1)))
    budget = int(args.budget_gib * (1 << 30))
    seed = 20260421
    t0 = time.time()
    q, k, v = (cqs_synth.torch_tensor((1, H, Np, D), seed, nm, torch.bfloat16, "cuda").cpu()
               .pin_memory() for nm in ("q", "k", "v"))
    torch.cuda.empty_cache()
    gen_s = time.time() - t0
    desc = dict(N=Np, B=1, H=H, D=D, depth=1, budget_bytes=budget, in_dtype="bf16",
                qkv_loc="host", out_loc="host")
    plan = cqs.cqs_plan(**desc)
    info = plan.info()
    dev, host = cqs.cqs_forward_workspace_size(plan)
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    ws = torch.empty(max(dev, 256), dtype=torch.uint8, device="cuda")
    hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
    out = torch.empty((1, H, Np, D), dtype=torch.bfloat16).pin_memory()
    lse = torch.empty((1, H, Np), dtype=torch.float32).pin_memory()
    # warm-up on a small problem (kernel attributes, TMA descriptors)
    cqs.attention(*(t[:, :, :4096].cuda() for t in (q, k, v)), depth=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = cqs.cqs_attention_forward(plan, q, k, v, out, lse, 0.0, budget, ws, hws, stats=True)
    e1.record()
    torch.cuda.synchronize()
    t7 = e0.elapsed_time(e1) / 1e3
    peak = torch.cuda.max_memory_allocated() - base
    useful = 4.0 * Np * Np * D * H
    rate = useful / t7
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(Np, args.rows, replace=False))
    kk = k[0, 0].double().numpy()
    vv = v[0, 0].double().numpy()
    Oref, lref = R.rows_forward(q[0, 0].double().numpy(), kk, vv, rows, block=1 << 20)
    o = out[0, 0, rows].double().numpy()
    l_ = lse[0, 0, rows].double().numpy()
    res = {
        "config": "C5 scaled evaluation (P:206): N'=%d = 1e9*(3/7)^%d, H=1, D=64, bf16, depth 1 "
                  "-> 7 leaves of the itr=%d tree, QKV/O in pinned host memory" % (
                      Np, args.itr - 1, args.itr),
        "t7_s": t7, "useful_tflops": rate / 1e12, "tokens": Np,
        "budget_bytes": budget, "predicted_peak_bytes": info.predicted_peak_bytes,
        "measured_peak_dev_bytes": peak, "acc_depth": info.acc_depth,
        "stage_buffers": info.n_stage_buffers, "bytes_h2d": st.bytes_h2d, "bytes_d2h": st.bytes_d2h,
        "h2d_gbs": st.bytes_h2d / t7 / 1e9,
        "est_1B_hours_paper_method": t7 * 7 ** (args.itr - 1) / 3600,
        "est_1B_hours_by_work": 4.0 * N_full ** 2 * D / rate / 3600,
        "paper_1B_fwd_A100_hours_itr%d" % args.itr: {5: 9510, 6: 12138, 7: 15621, 8: 20817,
                                                      9: 28824}.get(args.itr),
        "parity_rows": int(len(rows)), "max_abs_err": float(np.abs(o - Oref).max()),
        "max_lse_err": float(np.abs(l_ - lref).max()), "gen_s": gen_s,
    }
    if not args.no_bwd:
        res["backward"] = backward(args, q, k, v, out, lse, Np, H, D, N_full, seed)
    print(json.dumps(res))


def backward(args, q, k, v, out, lse, Np, H, D, N_full, seed):
    """Table 1's backward half (t7_bwd): Algorithm 2 on the same 7 leaves, STREAMED like the
    forward: Q, K, V, O, dO, lse and the gradients in pinned host memory, the fp32 gradient
    accumulators of all N' rows plus one or two staging buffers on the device, under the same
    16 GiB budget."""
    import numpy as np
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from tools import _rowref as R
    budget = int(args.budget_gib * (1 << 30))
    do = cqs_synth.torch_tensor((1, H, Np, D), seed, "do", torch.bfloat16, "cuda").cpu().pin_memory()
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dq, dk, dv, info, st = cqs.attention_backward_streamed(q, k, v, out, do, lse, depth=1,
                                                           budget_bytes=budget,
                                                           grad_dtype=torch.float32, stats=True)
    e1.record()
    torch.cuda.synchronize()
    t7 = e0.elapsed_time(e1) / 1e3
    peak = torch.cuda.max_memory_allocated() - base
    useful = 10.0 * Np * Np * D * H
    rate = useful / t7
    # invariants at any size: sum_j dV_j = sum_i dO_i (rows of P sum to 1); sum_j dK_j = 0
    s_dv, s_do = dv.double().sum(dim=2), do.double().sum(dim=2)
    inv_dv = float((s_dv - s_do).norm() / s_do.norm())
    inv_dk = float(dk.double().sum(dim=2).norm() / dk.double().norm())
    rng = np.random.default_rng(6)
    rows = np.sort(rng.choice(Np, 4, replace=False))
    f = lambda t: t[0, 0].double().numpy()
    ref = R.rows_dq(f(q), f(k), f(v), f(do), rows, block=1 << 20)
    got = dq[0, 0, rows].double().numpy()
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    return {"t7_bwd_s": t7, "useful_tflops_algorithmic": rate / 1e12, "mode": "streamed",
            "budget_bytes": budget, "workspace_bytes": info["workspace_bytes"],
            "measured_peak_dev_bytes": peak, "bytes_h2d": st.bytes_h2d, "bytes_d2h": st.bytes_d2h,
            "est_1B_bwd_hours_paper_method": t7 * 7 ** (args.itr - 1) / 3600,
            "est_1B_bwd_hours_by_work": 10.0 * N_full ** 2 * D / rate / 3600,
            "paper_1B_bwd_A100_hours_itr%d" % args.itr: {5: 23411, 6: 30075, 7: 38497, 8: 50556,
                                                          9: 67256}.get(args.itr),
            "paper_mem_bwd_GiB_itr%d" % args.itr: {5: 41.79, 6: 17.93, 7: 7.68, 8: 3.32,
                                                    9: 1.43}.get(args.itr),
            "parity_dq_rows": int(len(rows)), "max_dq_row_rel_err": float(rel.max()),
            "invariant_sum_dV_minus_sum_dO_rel": inv_dv, "invariant_sum_dK_rel": inv_dk}


if __name__ == "__main__":
    main()

"""BASELINE config 4 (C5) by SURVEY §8d's protocol: N = 1e9 tokens, 1 head, D = 64, bf16, Q/K/V in
host memory streamed through one B200, depth chosen by the memory model from the device budget.

The box has ~196 GB of RAM and the 1e9-token Q/K/V alone are 384 GB, so the buffers are REAL
1e9-token host address ranges (Q, K, V, O, lse and the pinned host accumulator: ~780 GB of virtual
memory, mmap MAP_NORESERVE) of which only the pages a batch of leaves touches are materialised
(by the seeded generator), page-locked (cudaHostRegister) and released after the batch.  Every
call goes through the public C ABI (cqs_plan with CQS_PLAN_SUBSET + cqs_attention_forward,
qkv_loc = out_loc = pinned host) exactly as a full pass would, streaming each task's segments H2D.

  (a) a work-weighted random sample of >= 64 non-empty leaves, run in DFS order in batches;
  (b) one contiguous DFS window (all leaves of one depth-(k-2) subtree: 49 leaves) — overlap of
      copies / compute / host-tier flushes over consecutive leaves;
  rate = useful FLOPs (4 D x kept pairs of the leaves run) / device time; the full pass is
  extrapolated by work: t = 4 N^2 D / rate (the paper extrapolates from t7 the same way).
Parity (per batch): sampled query rows of the leaves run; each equals the softmax over the union of
its kept key segments in those leaves (key sets from the plan's task table, which tests pin to the
literal Algorithm 3), computed in fp64 by tools/_rowref.py from the same host buffers.

    python tools/c5_protocol.py [--sample 64] [--window 49] [--budget-gib 16] > profiles/r02_c5.json
"""
import argparse
import ctypes
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAGE = 4096
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                      ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
libc.munmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t]


def vmap(nbytes):
    """Anonymous MAP_NORESERVE mapping: address space only, pages appear when touched."""
    addr = libc.mmap(None, nbytes, 3, 0x22 | 0x4000, -1, 0)
    if addr in (None, ctypes.c_void_p(-1).value):
        raise OSError(ctypes.get_errno(), "mmap failed")
    return addr


def as_tensor(addr, shape, dtype):
    import numpy as np
    import torch
    n = 1
    for s in shape:
        n *= s
    esz = {torch.bfloat16: 2, torch.float32: 4, torch.uint8: 1}[dtype]
    raw = np.ctypeslib.as_array((ctypes.c_uint8 * (n * esz)).from_address(addr))
    t = torch.from_numpy(raw)
    return t.view(dtype).view(*shape)


def page_union(ranges):
    """Byte ranges -> sorted disjoint page-aligned (start, len) ranges."""
    iv = sorted((a // PAGE * PAGE, (b + PAGE - 1) // PAGE * PAGE) for a, b in ranges if b > a)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return [(a, b - a) for a, b in out]


def row_union(ranges):
    iv = sorted((a, a + n) for a, n in ranges if n > 0)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return [(a, b - a) for a, b in out]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=10 ** 9)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--sample", type=int, default=64)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--window", type=int, default=49, help="0 = skip the contiguous window")
    ap.add_argument("--rows", type=int, default=2, help="parity rows per batch")
    ap.add_argument("--first-batch", type=int, default=0,
                    help="run the sample from this batch index on (resume a cut-off run: the "
                         "sample is seeded, so batches are reproducible)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from tools import _rowref as R

    N, H, D, seed = args.N, 1, 64, 20260421
    budget = int(args.budget_gib * (1 << 30))
    cudart = torch.cuda.cudart()
    res = {"config": "C5: N=%d, H=1, D=64, bf16, Q/K/V/O in host memory (MAP_NORESERVE 1e9-token "
                     "buffers, touched pages materialised + page-locked per batch), %.0f GiB device "
                     "budget" % (N, args.budget_gib)}
    with open("/proc/meminfo") as f:
        res["host_mem_total_gb"] = int(f.readline().split()[1]) / 1e6
    t0 = time.time()
    desc = dict(N=N, B=1, H=H, D=D, depth=-1, budget_bytes=budget, in_dtype="bf16",
                qkv_loc="host", out_loc="host")
    plan = cqs.cqs_plan(**desc)
    info = plan.info()
    k = info.depth
    nt = info.n_tasks
    works = np.array([plan.task(i).work for i in range(nt)], dtype=np.float64)
    res["plan"] = {"depth": k, "acc_depth": info.acc_depth, "stage_buffers": info.n_stage_buffers,
                   "tasks": nt, "empty": int(info.n_empty), "max_staged_rows": info.max_staged_rows,
                   "predicted_peak_bytes": info.predicted_peak_bytes,
                   "host_workspace_bytes": info.host_workspace_bytes,
                   "max_over_mean_work": float(works.max() / works[works > 0].mean()),
                   "plan_s": time.time() - t0}
    # virtual host buffers
    e = 2
    sz = {"q": N * D * e, "k": N * D * e, "v": N * D * e, "o": N * D * e, "l": N * 4,
          "hws": info.host_workspace_bytes}
    base = {nm: vmap(b) for nm, b in sz.items()}
    q, kk, v, o = (as_tensor(base[nm], (1, 1, N, D), torch.bfloat16) for nm in ("q", "k", "v", "o"))
    lse = as_tensor(base["l"], (1, 1, N), torch.float32)
    hws = as_tensor(base["hws"], (max(sz["hws"], 256),), torch.uint8)
    # the host accumulator's lse rows (all N are initialised by every call) and the output lse
    # stay page-locked for the whole run: 4 GB each
    hacc_l_off = (N * D * 4 + 255) // 256 * 256
    always = [(base["hws"] + hacc_l_off, N * 4), (base["l"], N * 4)]
    for a, n in always:
        assert int(cudart.cudaHostRegister(a, n, 0)) == 0
    dev = torch.device("cuda")
    dv, _ = cqs.cqs_forward_workspace_size(plan)
    torch.cuda.reset_peak_memory_stats()
    ws = torch.empty(dv, dtype=torch.uint8, device=dev)
    # warm-up (module loading) on a small problem
    cqs.attention(*(cqs_synth.torch_qkv(1, 1, 4096, D, 1, torch.bfloat16, "cuda")), depth=1)
    torch.cuda.synchronize()

    def task_rows(t):
        T = plan.task(int(t))
        used = set()
        for a in range(T.nseg):
            if T.kept[a]:
                used.add(a)
                used.update(b for b in range(T.nseg) if T.kept[a] >> b & 1)
        segs = [(T.seg_start[a], T.seg_len[a]) for a in range(T.nseg)]
        return T, segs, [segs[a] for a in sorted(used)]

    def run(tasks, label, rng):
        """One subset call over `tasks` (DFS order): materialise + lock the touched pages, run,
        check sampled rows, release."""
        tasks = sorted(int(t) for t in tasks)
        info_t = [task_rows(t) for t in tasks]
        qkv_rows = row_union([s for _, _, used in info_t for s in used])
        all_rows = row_union([s for _, segs, _ in info_t for s in segs])
        ranges = []
        for nm in ("q", "k", "v"):
            ranges += [(base[nm] + a * D * e, base[nm] + (a + n) * D * e) for a, n in qkv_rows]
        ranges += [(base["o"] + a * D * e, base["o"] + (a + n) * D * e) for a, n in all_rows]
        ranges += [(base["hws"] + a * D * 4, base["hws"] + (a + n) * D * 4) for a, n in all_rows]
        pages = page_union(ranges)
        t_reg = time.time()
        for a, n in pages:
            rc = int(cudart.cudaHostRegister(a, n, 0))
            assert rc == 0, "cudaHostRegister %d" % rc
        t_reg = time.time() - t_reg
        t_gen = time.time()
        for nm, tid in (("q", 0), ("k", 1), ("v", 2)):
            dst = {"q": q, "k": kk, "v": v}[nm]
            for a, n in qkv_rows:
                for s0 in range(a, a + n, 1 << 22):
                    c = min(1 << 22, a + n - s0)
                    dst[0, 0, s0:s0 + c].view(-1).copy_(cqs_synth.torch_values(
                        seed, tid, s0 * D, c * D, "cuda").to(torch.bfloat16))
        torch.cuda.synchronize()
        t_gen = time.time() - t_gen
        p = cqs.cqs_plan(exec_order=tasks, subset=True, **desc)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()   # the call's own bytes, not the generator's
        a0 = torch.cuda.memory_allocated()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = cqs.cqs_attention_forward(p, q, kk, v, o, lse, 0.0, budget, ws, hws, stats=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        call_peak = torch.cuda.max_memory_allocated() - a0 + ws.numel()
        work = float(sum(T.work for T, _, _ in info_t))
        # parity rows: query rows of active segments; reference over the union of their kept keys
        errs, lerrs = [], []
        for _ in range(args.rows):
            T, segs, _ = info_t[int(rng.integers(len(info_t)))]
            act = [a for a in range(T.nseg) if T.kept[a]]
            a = act[int(rng.integers(len(act)))]
            row = int(segs[a][0] + rng.integers(segs[a][1]))
            keys = []
            for T2, segs2, _ in info_t:
                for x in range(T2.nseg):
                    if T2.kept[x] and segs2[x][0] <= row < segs2[x][0] + segs2[x][1]:
                        keys += [segs2[y] for y in range(T2.nseg) if T2.kept[x] >> y & 1]
            idx = np.concatenate([np.arange(s, s + n) for s, n in keys])
            kr = kk[0, 0, idx].double().numpy()
            vr = v[0, 0, idx].double().numpy()
            Oref, lref = R.rows_forward(q[0, 0, row:row + 1].double().numpy(), kr, vr, [0],
                                        block=1 << 20)
            errs.append(float(np.abs(o[0, 0, row].double().numpy() - Oref[0]).max()))
            lerrs.append(float(abs(float(lse[0, 0, row]) - lref[0])))
        for a, n in pages:
            cudart.cudaHostUnregister(a)
            libc.madvise(a, n, 4)      # MADV_DONTNEED: give the pages back
        r = {"label": label, "tasks": len(tasks), "first_task": tasks[0], "last_task": tasks[-1],
             "useful_flop": 4.0 * D * work, "ms": ms, "tflops": 4.0 * D * work / (ms * 1e-3) / 1e12,
             "bytes_h2d": st.bytes_h2d, "bytes_d2h": st.bytes_d2h,
             "h2d_gbs_avg": st.bytes_h2d / (ms * 1e-3) / 1e9,
             "kernel_launches": st.kernel_launches, "host_gb_touched": sum(n for _, n in pages) / 1e9,
             "device_bytes_during_call": call_peak,
             "register_s": t_reg, "generate_s": t_gen,
             "parity_max_abs_err": max(errs), "parity_max_lse_err": max(lerrs),
             "parity_ok": max(errs) <= 2e-2 and max(lerrs) <= 1e-3}
        print(json.dumps(r), file=sys.stderr, flush=True)
        return r

    rng = np.random.default_rng(seed)
    nonempty = np.nonzero(works > 0)[0]
    pick = rng.choice(nonempty, size=min(args.sample, len(nonempty)), replace=False,
                      p=works[nonempty] / works[nonempty].sum())
    pick = np.sort(pick)
    batches = []
    for i in range(args.first_batch * args.batch, len(pick), args.batch):
        batches.append(run(pick[i:i + args.batch], "sample batch %d" % (i // args.batch),
                           np.random.default_rng(seed + 1 + i // args.batch)))
    res["sample"] = batches
    s_flop = sum(b["useful_flop"] for b in batches)
    s_ms = sum(b["ms"] for b in batches)
    rate = s_flop / (s_ms * 1e-3) if batches else float("nan")
    res["sample_rate_tflops"] = rate / 1e12
    if args.window:
        # all leaves under one depth-(k-2) node (49 leaves when k >= 2), DFS-contiguous; chosen at
        # random among the nodes whose leaves are all non-empty-ish (any node is valid)
        span = 7 ** 2 if k >= 2 else nt
        n0 = int(rng.integers(nt // span)) * span
        win = [t for t in range(n0, n0 + span) if works[t] > 0][:args.window]
        res["window"] = run(win, "window: tasks %d..%d" % (n0, n0 + span - 1),
                            np.random.default_rng(seed + 999))
    total_flop = 4.0 * N * N * D * H
    res["extrapolated_full_pass_h"] = total_flop / rate / 3600 if batches else None
    if args.window:
        res["extrapolated_full_pass_h_window_rate"] = total_flop / (
            res["window"]["tflops"] * 1e12) / 3600
    res["peak_device_bytes_allocator"] = torch.cuda.max_memory_allocated()
    res["budget_bytes"] = budget
    res["parity_ok"] = all(b["parity_ok"] for b in batches) and (
        not args.window or res["window"]["parity_ok"])
    res["wall_s"] = time.time() - t0
    print(json.dumps(res))


if __name__ == "__main__":
    main()

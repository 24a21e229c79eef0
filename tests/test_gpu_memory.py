"""Peak device memory against the budget, measured on the device (SURVEY §8c "O5 ... The measured
GPU peak must be <= budget and within about 10% of the predicted value"; PAPER.md P:146, P:162,
P:208).  This is the independent pin of the memory model (oracle/memory_model.py restates the
accounting; these tests check it against what the hardware reports):

  allocator : torch.cuda.max_memory_allocated delta over the call — the caller's tensors and the
              workspace as separate allocations; must be <= budget with NO slack and equal the
              prediction (the model counts every tensor at the allocator's 512-byte granularity);
  driver    : cudaMemGetInfo free-memory drop with everything live (2 MiB pages, incl. anything the
              library or the runtime allocates during the call) — within 10% of the prediction;
  nvml      : device-wide used-memory peak sampled every ~2 ms during the call — within 10%.

Several (depth, accumulator tier, staging buffers) choices, resident and streamed, and the task
execution order permuted (any order is exact: Eq. 3 is associative and commutative, P:48-52,
P:136 "fully independent" tasks)."""
import threading
import time

import numpy as np
import pytest
import torch

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O
from cqs_test_tiers import planner_tier

pytestmark = pytest.mark.gpu
DEV = "cuda"


class NvmlPeak:
    def __enter__(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.get = lambda: pynvml.nvmlDeviceGetMemoryInfo(h).used
        self.base = self.peak = self.get()
        self.stop = False

        def run():
            while not self.stop:
                self.peak = max(self.peak, self.get())
                time.sleep(0.002)

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.t.join()
        self.peak = max(self.peak, self.get())


def measured_call(alloc_and_run):
    """Run alloc_and_run() (allocates the call's device tensors, runs it, returns them) with the
    three measurements around it.  Returns (allocator, driver, nvml) bytes."""
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    a0 = torch.cuda.memory_allocated()
    free0 = torch.cuda.mem_get_info()[0]
    with NvmlPeak() as nv:
        keep = alloc_and_run()
        torch.cuda.synchronize()
        free1 = torch.cuda.mem_get_info()[0]
    alloc = torch.cuda.max_memory_allocated() - a0
    del keep
    torch.cuda.empty_cache()
    return alloc, free0 - free1, nv.peak - nv.base


def _warm(streamed, D):
    """Load the kernels' modules (lazy loading takes device memory at the first launch) before
    measuring."""
    q, k, v = cqs_synth.torch_qkv(1, 1, 3000, D, 1, dtype=torch.bfloat16,
                                  device="cpu" if streamed else DEV)
    if streamed:
        cqs.attention_streamed(q.pin_memory(), k.pin_memory(), v.pin_memory())
    else:
        cqs.attention(q, k, v, depth=2)
    torch.cuda.synchronize()


def check(pred, budget, alloc, drv, nv, n_tensors=1):
    assert pred <= budget
    assert alloc <= budget, (alloc, budget)                 # no slack
    # the model counts each tensor >= 1 MiB as whole 2 MiB pages (R14); torch's allocator reports
    # the 512-byte-rounded block when it splits a segment, the whole segment when it does not
    assert pred - (2 << 20) * n_tensors <= alloc <= pred, (alloc, pred)
    assert abs(drv - pred) <= 0.10 * pred, (drv, pred)
    assert abs(nv - pred) <= 0.10 * pred, (nv, pred)


@pytest.mark.parametrize("D", [128, 64])
def test_resident_bytes_measured(D):
    B, H, N = 1, 8, 65536
    _warm(False, D)
    q0, k0, v0 = cqs_synth.torch_qkv(B, H, N, D, 77, dtype=torch.bfloat16, device="cpu")
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=1)
    pred = p.info().predicted_peak_bytes
    dev, _ = cqs.cqs_forward_workspace_size(p)

    def run():
        q, k, v = (t.to(DEV) for t in (q0, k0, v0))
        out = torch.empty_like(q)
        lse = torch.empty(B, H, N, dtype=torch.float32, device=DEV)
        ws = torch.empty(dev, dtype=torch.uint8, device=DEV)
        cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, pred, ws, None)
        return q, k, v, out, lse, ws

    alloc, drv, nv = measured_call(run)
    check(pred, pred, alloc, drv, nv, n_tensors=6)


@pytest.mark.parametrize("depth,acc_depth,nbuf", [(1, 0, 2), (2, 0, 2), (2, 1, 2), (2, 2, 1),
                                                  (3, 1, 2), (3, 3, 1)])
def test_streamed_tiers_measured(depth, acc_depth, nbuf):
    """Streamed plans at several memory tiers, each given exactly its predicted bytes as the
    budget: the planner must pick the first fitting tier in its search order and the
    device must not use more."""
    B, H, N, D = 1, 8, 200000, 128
    _warm(True, D)
    q, k, v = (cqs_synth.torch_tensor((B, H, N, D), 78, nm, torch.bfloat16, DEV).cpu().pin_memory()
               for nm in ("q", "k", "v"))
    d = cqs.make_desc(N=N, B=B, H=H, D=D, depth=depth, in_dtype="bf16", qkv_loc="host")
    budget, _ = cqs.cqs_memory_model(d, depth, acc_depth, nbuf)
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget, in_dtype="bf16",
                     qkv_loc="host", out_loc="host")
    info = p.info()
    assert (info.depth, info.acc_depth, info.n_stage_buffers) == planner_tier(d, budget, [depth])
    dev, host = cqs.cqs_forward_workspace_size(p)
    hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
    out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
    lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()

    def run():
        ws = torch.empty(dev, dtype=torch.uint8, device=DEV)
        cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, budget, ws, hws)
        return ws

    alloc, drv, nv = measured_call(run)
    check(info.predicted_peak_bytes, budget, alloc, drv, nv)
    rows = np.array([0, 1, 77777, N // 2, N - 1])
    for h in (0, H - 1):
        Oref, lref = O.dense_attention_rows(*(t[0, h].double().numpy() for t in (q, k, v)), rows)
        assert np.abs(out[0, h, rows].double().numpy() - Oref).max() <= 2e-2
        assert np.abs(lse[0, h, rows].double().numpy() - lref).max() <= 1e-3


def test_budget_chosen_depth_measured():
    """depth = -1: the planner picks the smallest depth that fits; the measured bytes stay within
    the budget (C3-like shape scaled down to leave the test fast)."""
    B, H, N, D = 1, 16, 300000, 128
    budget = 1 << 30
    _warm(True, D)
    q, k, v = (cqs_synth.torch_tensor((B, H, N, D), 79, nm, torch.bfloat16, DEV).cpu().pin_memory()
               for nm in ("q", "k", "v"))
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=-1, budget_bytes=budget, in_dtype="bf16",
                     qkv_loc="host", out_loc="host")
    info = p.info()
    assert info.depth >= 1 and info.predicted_peak_bytes <= budget
    dev, host = cqs.cqs_forward_workspace_size(p)
    hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
    out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
    lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()

    def run():
        ws = torch.empty(dev, dtype=torch.uint8, device=DEV)
        cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, budget, ws, hws)
        return ws

    alloc, drv, nv = measured_call(run)
    check(info.predicted_peak_bytes, budget, alloc, drv, nv)
    assert drv <= budget and nv <= budget


@pytest.mark.parametrize("mode", ["resident", "streamed_j0", "streamed_j1"])
def test_task_order_permutation(mode):
    """A random execution order of the tasks gives the same attention (within the bf16 tolerance
    of the oracle, and within fp rounding of the lexicographic order)."""
    B, H, N, D = 1, 2, 3000, 128
    depth = 2
    q, k, v = cqs_synth.torch_qkv(B, H, N, D, 80, dtype=torch.bfloat16)
    perm = np.random.default_rng(5).permutation(7 ** depth)
    res = []
    for order in (None, perm):
        if mode == "resident":
            p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=depth, exec_order=order)
            qd, kd, vd = (t.to(DEV) for t in (q, k, v))
            ws = torch.empty(cqs.cqs_forward_workspace_size(p)[0], dtype=torch.uint8, device=DEV)
            out = torch.empty_like(qd)
            lse = torch.empty(B, H, N, dtype=torch.float32, device=DEV)
            cqs.cqs_attention_forward(p, qd, kd, vd, out, lse, 0.0, 0, ws, None)
        else:
            j = 0 if mode == "streamed_j0" else 1
            d = cqs.make_desc(N=N, B=B, H=H, D=D, depth=depth, in_dtype="bf16", qkv_loc="host")
            budget, _ = cqs.cqs_memory_model(d, depth, j, 2)
            p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget,
                             in_dtype="bf16", qkv_loc="host", out_loc="host", exec_order=order)
            assert p.info().acc_depth == planner_tier(d, budget, [depth])[1]
            dv, hb = cqs.cqs_forward_workspace_size(p)
            ws = torch.empty(dv, dtype=torch.uint8, device=DEV)
            hws = torch.empty(max(hb, 256), dtype=torch.uint8).pin_memory() if hb else None
            qh, kh, vh = (t.pin_memory() for t in (q, k, v))
            out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
            lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()
            cqs.cqs_attention_forward(p, qh, kh, vh, out, lse, 0.0, 0, ws, hws)
        torch.cuda.synchronize()
        res.append((out.double().cpu().numpy(), lse.double().cpu().numpy()))
    Oref, lref = O.dense_attention(*(t.double().numpy() for t in (q, k, v)))
    for o, l_ in res:
        assert np.abs(o - Oref).max() <= 2e-2 and np.abs(l_ - lref).max() <= 1e-3
    assert np.abs(res[0][0] - res[1][0]).max() <= 1e-2
    assert np.abs(res[0][1] - res[1][1]).max() <= 1e-5

"""GPU parity of the streamed path (Q/K/V and O/lse in pinned host memory, staged per task; DESIGN.md
"Streamed executor") against the fp64 oracle, and peak device memory against the budget."""
import numpy as np
import pytest
import torch

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O
from cqs_test_tiers import planner_tier

pytestmark = pytest.mark.gpu


def host_qkv(B, H, N, D, seed, dt):
    return tuple(t.pin_memory() for t in cqs_synth.torch_qkv(B, H, N, D, seed, dtype=dt))


def run_streamed(q, k, v, budget, depth=-1, out_dtype=None):
    B, H, N, D = q.shape
    ind = "bf16" if q.dtype == torch.bfloat16 else "f32"
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget, in_dtype=ind,
                     out_dtype=out_dtype or ind, qkv_loc="host", out_loc="host")
    info = p.info()
    dev, host = cqs.cqs_forward_workspace_size(p)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    ws = torch.empty(max(dev, 256), dtype=torch.uint8, device="cuda")
    hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
    odt = q.dtype if out_dtype is None else {"bf16": torch.bfloat16, "f32": torch.float32}[out_dtype]
    out = torch.empty(q.shape, dtype=odt).pin_memory()
    lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()
    st = cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, budget, ws, hws, stats=True)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    return out, lse, info, st, peak


def check(out, lse, q, k, v, tol_o, tol_l):
    Oref, lref = O.dense_attention(*(t.double().numpy() for t in (q, k, v)))
    err = np.abs(out.double().numpy() - Oref)
    assert err.max() <= tol_o and err.max() / np.abs(Oref).max() <= tol_o, err.max()
    assert np.abs(lse.double().numpy() - lref).max() <= tol_l


@pytest.mark.parametrize("N,H,D", [(3000, 2, 128), (2500, 2, 64)])
def test_streamed_bf16_budget_tiers(N, H, D):
    q, k, v = host_qkv(1, H, N, D, 31 + N, torch.bfloat16)
    d = cqs.make_desc(N=N, B=1, H=H, D=D, depth=-1, in_dtype="bf16", qkv_loc="host")
    # (depth, budget tier) -> the exact tier the planner must pick (DESIGN §8 search order)
    for (kk, j, nb, unlimited) in [(2, 1, 2, False), (1, 0, 2, True), (2, 2, 1, False),
                                   (3, 2, 2, False)]:
        budget = 0 if unlimited else cqs.cqs_memory_model(d, kk, j, nb)[0]
        out, lse, info, st, peak = run_streamed(q, k, v, budget, depth=kk)
        want = (kk, j, nb) if unlimited else planner_tier(d, budget, [kk])
        assert (info.depth, info.acc_depth, info.n_stage_buffers) == want
        budget = budget or info.predicted_peak_bytes
        # peak through torch's allocator: the model counts every tensor at its 512-byte granularity
        assert info.predicted_peak_bytes <= budget and peak <= budget
        assert st.bytes_h2d > 0 and st.tasks_run == info.my_tasks
        check(out, lse, q, k, v, 2e-2, 1e-3)


def test_streamed_f32():
    q, k, v = host_qkv(1, 1, 1030, 64, 5, torch.float32)
    d = cqs.make_desc(N=1030, B=1, H=1, D=64, depth=-1, in_dtype="f32", qkv_loc="host")
    budget, _ = cqs.cqs_memory_model(d, 2, 1, 2)
    out, lse, info, st, peak = run_streamed(q, k, v, budget)
    assert info.depth == 2 and info.acc_depth == 1
    check(out, lse, q, k, v, 1e-5, 1e-5)


@pytest.mark.slow
def test_c3_streamed_16gib_sampled():
    """BASELINE config 2: N=1M, H=32, D=128, bf16, QKV in pinned host, 16 GiB budget -> depth 2;
    peak device bytes <= budget; sampled rows vs the oracle."""
    B, H, N, D = 1, 32, 1_000_000, 128
    budget = 16 << 30
    # generated on the GPU (same integers as the CPU generator), kept in pinned host memory
    q, k, v = (cqs_synth.torch_tensor((B, H, N, D), 20260419, nm, torch.bfloat16, "cuda")
               .cpu().pin_memory() for nm in ("q", "k", "v"))
    torch.cuda.empty_cache()
    out, lse, info, st, peak = run_streamed(q, k, v, budget)
    assert info.depth == 2 and peak <= budget
    rng = np.random.default_rng(2)
    # 4 heads x 64 rows: random rows plus the first / last token and both sides of every level-1
    # and level-2 chunk boundary (BalancedChunkLayout, R1)
    edges = []
    for c in (7, 49):
        base, rem = divmod(N, c)
        b = np.cumsum([base + (i < rem) for i in range(c)])[:-1]
        edges += list(b - 1) + list(b)
    for h in rng.choice(H, 4, replace=False):
        pick = rng.choice(edges, 24, replace=False)
        rows = np.unique(np.concatenate([[0, N - 1], pick, rng.choice(N, 38, replace=False)]))
        Oref, lref = O.dense_attention_rows(q[0, h].double().numpy(), k[0, h].double().numpy(),
                                            v[0, h].double().numpy(), rows, block=65536)
        o = out[0, h, rows].double().numpy()
        assert np.abs(o - Oref).max() <= 2e-2
        assert np.abs(lse[0, h, rows].double().numpy() - lref).max() <= 1e-3


def test_streamed_batch2_f32_out():
    q, k, v = host_qkv(2, 2, 1500, 128, 77, torch.bfloat16)
    d = cqs.make_desc(N=1500, B=2, H=2, D=128, depth=-1, in_dtype="bf16", qkv_loc="host")
    budget, _ = cqs.cqs_memory_model(d, 2, 1, 1)
    out, lse, info, st, peak = run_streamed(q, k, v, budget, depth=2, out_dtype="f32")
    assert info.depth == 2 and peak <= budget
    check(out, lse, q, k, v, 2e-2, 1e-3)


def test_guardrail_retries_one_level_deeper():
    """OOM guardrail: a budget larger than what the device can actually give makes the
    workspace allocation fail; the call re-plans at itr + 1 and succeeds, matching the oracle."""
    import numpy as np
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from oracle import cqs_oracle as O
    B, H, N, D = 1, 4, 60000, 128
    q, k, v = (cqs_synth.torch_tensor((B, H, N, D), 61, nm, torch.bfloat16).pin_memory()
               for nm in ("q", "k", "v"))
    torch.cuda.synchronize()
    torch.cuda.empty_cache()    # cached blocks of earlier tests would otherwise satisfy the alloc
    free = torch.cuda.mem_get_info()[0]
    # leave ~600 MB free: the depth-0 plan needs ~740 MB of workspace; after calibration (free -
    # 256 MB reserve) depth 1 with a depth-1 accumulator tier needs ~320 MB
    blocker = torch.empty(int(free - (600 << 20)), dtype=torch.uint8, device="cuda")
    try:
        out, lse, info = cqs.attention_streamed(q, k, v, budget_bytes=1 << 40)
    finally:
        del blocker
        torch.cuda.empty_cache()
    assert info["attempts"] > 1 and info["depth"] >= 1
    rows = np.array([0, 4999, 12345, 59999])
    for h in range(H):
        Oref, lref = O.dense_attention_rows(q[0, h].double().numpy(), k[0, h].double().numpy(),
                                            v[0, h].double().numpy(), rows)
        assert np.abs(out[0, h, rows].double().numpy() - Oref).max() <= 2e-2
        assert np.abs(lse[0, h, rows].double().numpy() - lref).max() <= 1e-3


def test_guardrail_default_budget_from_free_memory():
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    q, k, v = (cqs_synth.torch_tensor((1, 2, 5000, 64), 62, nm, torch.bfloat16).pin_memory()
               for nm in ("q", "k", "v"))
    out, lse, info = cqs.attention_streamed(q, k, v)
    assert info["attempts"] == 1 and info["depth"] == 0 and torch.isfinite(out.float()).all()


def test_streamed_mixed_level_interest_sets():
    """Per-level interest sets in the streamed executor (staging + accumulator tier)."""
    import numpy as np
    import torch
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from oracle import cqs_oracle as O
    B, H, N, D = 1, 2, 3000, 128
    q, k, v = (cqs_synth.torch_tensor((B, H, N, D), 64, nm, torch.bfloat16).pin_memory()
               for nm in ("q", "k", "v"))
    levels = [(13, (0, 1, 3, 9)), (7, (0, 1, 3))]
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=2, in_dtype="bf16", qkv_loc="host",
                     out_loc="host", levels=levels)
    dev, host = cqs.cqs_forward_workspace_size(p)
    ws = torch.empty(max(dev, 256), dtype=torch.uint8, device="cuda")
    hws = torch.empty(max(host, 256), dtype=torch.uint8).pin_memory() if host else None
    out = torch.empty((B, H, N, D), dtype=torch.bfloat16).pin_memory()
    lse = torch.empty((B, H, N), dtype=torch.float32).pin_memory()
    cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, hws)
    torch.cuda.synchronize()
    Od, ld = O.dense_attention(*(t.double().numpy() for t in (q, k, v)))
    assert np.abs(out.double().numpy() - Od).max() <= 2e-2
    assert np.abs(lse.double().numpy() - ld).max() <= 1e-3


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("N,depth,nb", [(1, 0, 2), (300, 0, 2), (777, 1, 2), (2401, 2, 2),
                                        (1500, 3, 2)])
def test_streamed_device_tier_first_last_split(N, depth, nb, D):
    """Device-tier accumulator (j = 0): the first task runs segment by segment as its staging
    lands, the last task query segment by query segment, and every row is downloaded right after
    its last task — each launch LSE-merges a partial over a key subset, so the result must still
    equal dense attention; ragged sizes, depth 0 (a single task) to 3."""
    H = 2
    q, k, v = host_qkv(1, H, N, D, 91 + N + D, torch.bfloat16)
    d = cqs.make_desc(N=N, B=1, H=H, D=D, depth=-1, in_dtype="bf16", qkv_loc="host")
    budget = cqs.cqs_memory_model(d, depth, 0, nb)[0]
    out, lse, info, st, peak = run_streamed(q, k, v, budget, depth=depth)
    assert (info.depth, info.acc_depth, info.n_stage_buffers) == planner_tier(d, budget, [depth])
    assert info.acc_depth == 0
    assert peak <= budget
    check(out, lse, q, k, v, 2e-2, 1e-3)

"""GPU parity of the backward (Algorithm 2) through the C ABI against the fp64
oracle's dense attention gradients (oracle O6, pinned to finite differences in
tests/test_oracle_backward.py) on the same seeded bf16 inputs.

Tolerance (R19): P and dS enter the tensor-core products as bf16 (relative rounding
2^-9), O and dO are bf16; per gradient tensor ||G - R||_F / ||R||_F <= 1e-2 and per row
||G_r - R_r||_2 <= 3e-2 ||R_r||_2 + 1e-3 rms(R).
"""
import numpy as np
import pytest
import torch

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def inputs(B, H, N, D, seed):
    q, k, v = cqs_synth.torch_qkv(B, H, N, D, seed, dtype=torch.bfloat16, device=DEV)
    do = cqs_synth.torch_tensor((B, H, N, D), seed, "do", torch.bfloat16, DEV)
    return q, k, v, do


def check_grads(got, ref, name):
    g = got.double().cpu().numpy()
    err = g - ref
    rel = np.linalg.norm(err) / np.linalg.norm(ref)
    rms = np.sqrt(np.mean(ref ** 2))
    row_err = np.linalg.norm(err, axis=-1)
    row_ref = np.linalg.norm(ref, axis=-1)
    worst = (row_err / (3e-2 * row_ref + 1e-3 * rms)).max()
    assert np.isfinite(g).all(), name
    assert rel <= 1e-2, (name, rel)
    assert worst <= 1.0, (name, worst, rel)
    return rel


def run(q, k, v, do, depth, grad_dtype=torch.float32):
    out, lse = cqs.attention(q, k, v, depth=depth)
    return cqs.attention_backward(q, k, v, out, do, lse, depth=depth, grad_dtype=grad_dtype)


def ref(q, k, v, do):
    f = lambda t: t.double().cpu().numpy()
    return O.dense_attention_grads(f(q), f(k), f(v), f(do))


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("N,depth", [(1030, 1), (1030, 2), (2401, 3), (300, 0), (49, 1), (130, 1)])
def test_backward_matches_dense_gradients(N, depth, D):
    q, k, v, do = inputs(1, 2, N, D, 31 + N + D)
    grads = run(q, k, v, do, depth)
    torch.cuda.synchronize()
    for g, r, nm in zip(grads, ref(q, k, v, do), ("dQ", "dK", "dV")):
        check_grads(g, r, nm)


def test_backward_batched_strided_bf16_out():
    """B=2, H=3, [B,N,H,D] storage viewed as [B,H,N,D], bf16 gradients."""
    B, H, N, D = 2, 3, 777, 128
    q, k, v, do = inputs(B, H, N, D, 5)
    qs, ks, vs, dos = (t.transpose(1, 2).contiguous().transpose(1, 2) for t in (q, k, v, do))
    out, lse = cqs.attention(qs, ks, vs, depth=2)
    outs = out.transpose(1, 2).contiguous().transpose(1, 2)
    grads = cqs.attention_backward(qs, ks, vs, outs, dos, lse, depth=2, grad_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    for g, r, nm in zip(grads, ref(q, k, v, do), ("dQ", "dK", "dV")):
        check_grads(g, r, nm)


def test_backward_depth_invariance():
    """Sum over tasks is the dense gradient at every depth (R19): depth 1 and 3 agree."""
    q, k, v, do = inputs(1, 2, 2401, 64, 77)
    g1 = run(q, k, v, do, 1)
    g3 = run(q, k, v, do, 3)
    torch.cuda.synchronize()
    for a, b in zip(g1, g3):
        assert (a - b).norm() / b.norm() < 5e-3


def test_backward_sampled_rows_c2_shape():
    """Launch configuration of the backward bench (N=131072, H=32, D=128, depth 1): sampled dQ
    rows against the oracle's per-row gradient (dense_dq_rows); dK / dV through identities that
    hold at any size: sum_j dV_j = sum_i dO_i (rows of P sum to 1) and sum_j dK_j = 0 (rows of dS
    sum to 0)."""
    B, H, N, D = 1, 32, 131072, 128
    q, k, v, do = inputs(B, H, N, D, 20260418)
    out, lse = cqs.attention(q, k, v, depth=1)
    dq, dk, dv = cqs.attention_backward(q, k, v, out, do, lse, depth=1, grad_dtype=torch.float32)
    torch.cuda.synchronize()
    # invariant 1: sum_j dV_j = sum_i (sum_j P_ij) dO_i = sum_i dO_i
    s_dv = dv.double().sum(dim=2)
    s_do = do.double().sum(dim=2)
    assert ((s_dv - s_do).norm() / s_do.norm()).item() < 1e-3
    # invariant 2: sum_j dK_j = alpha sum_i sum_j dS_ij q_i = 0 since sum_j dS_ij = 0
    s_dk = dk.double().sum(dim=2)
    assert (s_dk.norm() / dk.double().norm()).item() < 1e-2
    # sampled rows of dQ against the oracle (full key range per row)
    rng = np.random.default_rng(3)
    for h in rng.choice(H, 2, replace=False):
        rows = np.sort(rng.choice(N, 4, replace=False))
        f = lambda t: t[0, h].double().cpu().numpy()
        dq_ref = O.dense_dq_rows(f(q), f(k), f(v), f(do), rows)
        got = dq[0, h, rows].double().cpu().numpy()
        rel = np.linalg.norm(got - dq_ref, axis=1) / np.linalg.norm(dq_ref, axis=1)
        assert rel.max() < 3e-2, rel


def test_backward_rejects_unsupported():
    p = cqs.cqs_plan(N=1000, B=1, H=1, D=64, depth=1, in_dtype="f32")
    with pytest.raises(cqs.CqsError):
        cqs.cqs_backward_workspace_size(p)


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("N,depth", [(3000, 1), (2401, 2), (700, 0)])
def test_streamed_backward_matches_dense_gradients(N, depth, D):
    """Host-resident Q/K/V/O/dO/lse and gradients: staged per task, same kernels (R19 bar)."""
    q, k, v, do = inputs(1, 2, N, D, 71 + N + D)
    out, lse = cqs.attention(q, k, v, depth=depth)
    hq, hk, hv, ho, hdo = (t.cpu().pin_memory() for t in (q, k, v, out, do))
    hl = lse.cpu().pin_memory()
    dq, dk, dv, info = cqs.attention_backward_streamed(hq, hk, hv, ho, hdo, hl, depth=depth,
                                                       grad_dtype=torch.float32)
    assert info["depth"] == depth
    for g, r, nm in zip((dq, dk, dv), ref(q, k, v, do), ("dQ", "dK", "dV")):
        check_grads(g, r, nm)


def test_streamed_backward_budget_one_staging_buffer():
    """A budget between the one- and two-buffer footprints selects one staging buffer; the
    measured device peak stays within the budget; results equal the resident backward."""
    B, H, N, D = 1, 4, 20000, 128
    q, k, v, do = inputs(B, H, N, D, 5)
    out, lse = cqs.attention(q, k, v, depth=1)
    res = cqs.attention_backward(q, k, v, out, do, lse, depth=1, grad_dtype=torch.float32)
    hq, hk, hv, ho, hdo = (t.cpu().pin_memory() for t in (q, k, v, out, do))
    hl = lse.cpu().pin_memory()
    p2 = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=1, in_dtype="bf16", out_dtype="f32",
                      qkv_loc="host", out_loc="host")
    two = cqs.cqs_backward_workspace_size(p2)
    stage_one = 4 * B * H * cqs.cqs_plan_info(p2).max_staged_rows * D * 2
    budget = two - stage_one // 2        # fits one staging buffer, not two
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    dq, dk, dv, info = cqs.attention_backward_streamed(hq, hk, hv, ho, hdo, hl, depth=1,
                                                       budget_bytes=budget,
                                                       grad_dtype=torch.float32)
    peak = torch.cuda.max_memory_allocated() - base
    assert info["workspace_bytes"] <= budget < two and peak <= budget
    for a, b in zip((dq, dk, dv), res):
        assert (a.cuda() - b).abs().max().item() <= 1e-6 * max(1.0, b.abs().max().item())

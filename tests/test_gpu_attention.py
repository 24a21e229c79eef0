"""GPU parity: libcqs (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances:
  fp32 path  : normwise max|O-R| / max|R| <= 1e-5 globally and per output row (R15)
  bf16 path  : max|O-R| <= 2e-2 (BASELINE), normwise <= 2e-2, |lse - lse_ref| <= 1e-3 (R16)
"""
import math

import numpy as np
import pytest
import torch

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O

pytestmark = pytest.mark.gpu
I = (0, 1, 3)
DEV = "cuda"


def gen(B, H, N, D, seed, bf16):
    dt = torch.bfloat16 if bf16 else torch.float32
    q, k, v = cqs_synth.torch_qkv(B, H, N, D, seed, dtype=dt, device=DEV)
    return q, k, v


def ref_dense(q, k, v):
    return O.dense_attention(q.double().cpu().numpy(), k.double().cpu().numpy(),
                             v.double().cpu().numpy())


def check_f32(out, lse, Oref, lref):
    o = out.double().cpu().numpy()
    err = np.abs(o - Oref)
    assert err.max() / np.abs(Oref).max() <= 1e-5, err.max()
    row_rel = err.max(axis=-1) / np.abs(Oref).max(axis=-1)
    assert row_rel.max() <= 1e-5, row_rel.max()
    assert np.abs(lse.double().cpu().numpy() - lref).max() <= 1e-5


def check_bf16(out, lse, Oref, lref):
    o = out.double().cpu().numpy()
    err = np.abs(o - Oref)
    assert err.max() <= 2e-2, err.max()
    assert err.max() / np.abs(Oref).max() <= 2e-2, err.max() / np.abs(Oref).max()
    assert np.abs(lse.double().cpu().numpy() - lref).max() <= 1e-3


@pytest.mark.parametrize("N,depth", [(448, 1), (448, 2), (343, 3), (1030, 3), (7, 1), (100, 0)])
def test_f32_matches_oracle(N, depth):
    """BASELINE config 0 (N=448, D=64, fp32, one level) plus deeper trees with fully-masked rows
    and empty tasks."""
    q, k, v = gen(1, 2, N, 64, 20260417 + N, bf16=False)
    out, lse = cqs.attention(q, k, v, depth=depth)
    torch.cuda.synchronize()
    check_f32(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("N,depth", [(1030, 1), (1030, 2), (2401, 3), (300, 0), (49, 1)])
def test_bf16_matches_oracle(N, depth, D):
    q, k, v = gen(1, 2, N, D, 7 + N + D, bf16=True)
    out, lse = cqs.attention(q, k, v, depth=depth)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


def test_bf16_multi_batch_strided():
    B, H, N, D = 2, 3, 777, 128
    q, k, v = gen(B, H, N, D, 99, bf16=True)
    # non-contiguous: [B,N,H,D] storage viewed as [B,H,N,D]
    qs, ks, vs = (t.transpose(1, 2).contiguous().transpose(1, 2) for t in (q, k, v))
    out, lse = cqs.attention(qs, ks, vs, depth=2, out_dtype=torch.float32)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


def test_bf16_large_logits_rescale():
    """Scaled inputs make the running max jump across tiles (exercises conditional rescale)."""
    q, k, v = gen(1, 1, 3000, 128, 5, bf16=True)
    q = (q.float() * 3).to(torch.bfloat16)
    out, lse = cqs.attention(q, k, v, depth=1)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


def test_needle_routing():
    """SURVEY §8d needle: a key whose chunk differs from the query's at every level gets logit ~12;
    the output row is then ~V[m], so a dropped / duplicated / misrouted block moves O by O(1)."""
    B, H, N, D = 1, 1, 4096, 128
    q, k, v = gen(B, H, N, D, 11, bf16=True)
    qf, kf, vf = q.float().clone(), k.float().clone(), v.float().clone()
    rng = np.random.default_rng(0)
    alpha = 1 / math.sqrt(D)
    for n in rng.choice(N, 16, replace=False):
        m = (n + N // 2 + 13) % N
        kf[0, 0, m] = qf[0, 0, n] * (12.0 / (alpha * float((qf[0, 0, n] ** 2).sum())))
        vf[0, 0, m] = torch.tensor([1.0 if (i * 7 + n) % 3 else -1.0 for i in range(D)])
    q, k, v = (t.to(torch.bfloat16) for t in (qf, kf, vf))
    for depth in (1, 2, 3):
        out, lse = cqs.attention(q, k, v, depth=depth)
        torch.cuda.synchronize()
        check_bf16(out, lse, *ref_dense(q, k, v))


def test_deterministic():
    q, k, v = gen(1, 4, 5000, 128, 3, bf16=True)
    a, la = cqs.attention(q, k, v, depth=2)
    b, lb = cqs.attention(q, k, v, depth=2)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(la, lb)


@pytest.mark.parametrize("D", [128, 64])
def test_c2_full_size_sampled_rows(D):
    """BASELINE config 1 at full size (N=131072, H=32, D=128, bf16, one level), launched exactly as
    bench.py does (and the same shape at C5's head dim D=64); 128 sampled (head, row) outputs
    against the oracle's blockwise dense rows."""
    B, H, N = 1, 32, 131072
    q, k, v = gen(B, H, N, D, 20260418, bf16=True)
    out, lse = cqs.attention(q, k, v, depth=1)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    for h in rng.choice(H, 4, replace=False):
        rows = np.sort(rng.choice(N, 32, replace=False))
        rows[0], rows[-1] = 0, N - 1
        kk = k[0, h].double().cpu().numpy()
        vv = v[0, h].double().cpu().numpy()
        qq = q[0, h].double().cpu().numpy()
        Oref, lref = O.dense_attention_rows(qq, kk, vv, rows, block=16384)
        o = out[0, h, torch.from_numpy(rows).to(DEV)].double().cpu().numpy()
        l_ = lse[0, h, torch.from_numpy(rows).to(DEV)].double().cpu().numpy()
        assert np.abs(o - Oref).max() <= 2e-2
        assert np.abs(o - Oref).max() / np.abs(Oref).max() <= 2e-2
        assert np.abs(l_ - lref).max() <= 1e-3


def test_merge_abi_matches_oracle():
    rows, B, H, D = 1000, 1, 3, 128
    g = torch.Generator().manual_seed(0)
    parts_o = [torch.randn(rows, B * H, D, generator=g) for _ in range(3)]
    parts_l = [torch.randn(rows, B * H, generator=g) * 3 for _ in range(3)]
    parts_l[1][::7] = -math.inf
    for t in parts_l:
        t[5] = -math.inf
    ref_o, ref_l = O.lse_merge([(po.double().numpy(), pl.double().numpy())
                                for po, pl in zip(parts_o, parts_l)])
    out = torch.empty(B, H, rows, D, device=DEV)
    lse = torch.empty(B, H, rows, device=DEV)
    cqs.cqs_merge(rows, B, H, D, [t.to(DEV) for t in parts_o], [t.to(DEV) for t in parts_l],
                  out=out, lse_out=lse)
    torch.cuda.synchronize()
    got_o = out.permute(2, 0, 1, 3).reshape(rows, B * H, D).double().cpu().numpy()
    got_l = lse.permute(2, 0, 1).reshape(rows, B * H).double().cpu().numpy()
    assert np.allclose(got_o, ref_o, atol=1e-5) and np.all(got_o[5] == 0)
    fin = np.isfinite(ref_l)
    assert np.allclose(got_l[fin], ref_l[fin], atol=1e-5) and np.all(np.isneginf(got_l[~fin]))


@pytest.mark.parametrize("D", [32, 96, 128])
def test_f32_head_dims(D):
    q, k, v = gen(1, 1, 700, D, 41 + D, bf16=False)
    out, lse = cqs.attention(q, k, v, depth=2)
    torch.cuda.synchronize()
    check_f32(out, lse, *ref_dense(q, k, v))


def test_bf16_out_f32_depth0_tiny():
    """N smaller than one tile, single task (depth 0), fp32 output."""
    q, k, v = gen(1, 3, 37, 64, 17, bf16=True)
    out, lse = cqs.attention(q, k, v, depth=0, out_dtype=torch.float32)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("D", [64, 128])
def test_bf16_growing_logits_speculative_max(D):
    """Key norms grow along the sequence, so later key tiles raise the row max by more than the
    rescale threshold: exercises the speculative-max redo path (O rescale + second exp pass)."""
    N = 3000
    q, k, v = gen(1, 2, N, D, 123 + D, bf16=True)
    ramp = torch.linspace(0.5, 4.0, N, device=DEV).view(1, 1, N, 1)
    k = (k.float() * ramp).to(torch.bfloat16)
    for depth in (0, 1, 2):
        out, lse = cqs.attention(q, k, v, depth=depth)
        torch.cuda.synchronize()
        check_bf16(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("c,I,N,depth", [(13, (0, 1, 3, 9), 2000, 1), (13, (0, 1, 3, 9), 3000, 2),
                                         (7, (0, 1, 5), 2500, 2), (21, (0, 1, 4, 14, 16), 3000, 1)])
def test_bf16_other_interest_sets(c, I, N, depth):
    """NEXT-3: the same kernels run CQS Divide with c=13 / 21 and the paired c=7 set (P:350,
    P:366-368); the decomposition must still reproduce full attention."""
    q, k, v = gen(1, 2, N, 128, 300 + c + N, bf16=True)
    out, lse = cqs.attention(q, k, v, depth=depth, offsets=I)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("levels,N,depth", [([(7, (0, 1, 3)), (13, (0, 1, 3, 9))], 3000, 2),
                                            ([(13, (0, 1, 3, 9)), (7, (0, 1, 5))], 2500, 2)])
def test_bf16_mixed_level_interest_sets(levels, N, depth):
    """NEXT-3: a different c per divide level through the same kernels."""
    q, k, v = gen(1, 2, N, 128, 500 + N, bf16=True)
    p = cqs.cqs_plan(N=N, B=1, H=2, D=128, depth=depth, in_dtype="bf16", levels=levels)
    dev, _ = cqs.cqs_forward_workspace_size(p)
    ws = torch.empty(dev, dtype=torch.uint8, device=DEV)
    out = torch.empty_like(q)
    lse = torch.empty((1, 2, N), dtype=torch.float32, device=DEV)
    cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, None)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("N,depth", [(1, 0), (2, 0), (7, 1), (127, 0), (128, 0), (129, 0),
                                     (255, 1), (256, 1), (257, 1), (511, 0), (512, 0), (513, 0),
                                     (1025, 1), (343, 3)])
def test_bf16_tile_boundaries(N, depth, D):
    """Ragged sizes around the kernels' tile and work-item edges (128-row tiles; 384-row items at
    D=64, 512-row CTA-pair items at D=128, where one CTA of the pair or one tile may hold no row
    of the segment), one to three heads, single-token chunks at depth 1/3."""
    H = 1 + N % 3
    q, k, v = gen(1, H, N, D, 900 + N + D, bf16=True)
    out, lse = cqs.attention(q, k, v, depth=depth)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("N,depth", [(95, 0), (96, 0), (97, 0), (191, 0), (192, 0), (193, 0),
                                     (383, 0), (384, 0), (385, 0), (769, 0), (672, 1), (679, 1),
                                     (2689, 1)])
def test_bf16_d64_three_tile_edges(N, depth):
    """D = 64 runs three 128-row tiles per CTA (384-row items) over 96-key K/V tiles: ragged sizes
    around the 96-key tile edges (a key segment's last tile with 1 / 95 / 96 valid keys), the
    384-row item edges (items holding 1, 2 or 3 tiles) and depth-1 chunks of 96 +- 1 rows."""
    H = 1 + N % 3
    q, k, v = gen(1, H, N, 64, 1900 + N, bf16=True)
    out, lse = cqs.attention(q, k, v, depth=depth)
    torch.cuda.synchronize()
    check_bf16(out, lse, *ref_dense(q, k, v))


@pytest.mark.parametrize("streamed", [False, True])
def test_subset_calls_merge_to_full_attention(streamed):
    """CQS_PLAN_SUBSET: the tree split over two calls (even / odd task indices), each call's
    (O, lse) the LSE merge of its tasks only; merging the two results with cqs_merge (Eq. 3,
    P:48-52) gives full attention."""
    B, H, N, D, depth = 1, 2, 2500, 128, 2
    q, k, v = gen(B, H, N, D, 2024, bf16=True)
    halves = [list(range(0, 49, 2)), list(range(1, 49, 2))]
    res = []
    for sub in halves:
        kw = dict(N=N, B=B, H=H, D=D, depth=depth, exec_order=sub, subset=True)
        if streamed:
            p = cqs.cqs_plan(qkv_loc="host", out_loc="host", out_dtype="f32", **kw)
            dv, hb = cqs.cqs_forward_workspace_size(p)
            ws = torch.empty(dv, dtype=torch.uint8, device=DEV)
            hws = torch.empty(max(hb, 256), dtype=torch.uint8).pin_memory() if hb else None
            out = torch.zeros(q.shape, dtype=torch.float32).pin_memory()
            lse = torch.full(q.shape[:3], -math.inf, dtype=torch.float32).pin_memory()
            qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
            cqs.cqs_attention_forward(p, qh, kh, vh, out, lse, 0.0, 0, ws, hws)
        else:
            p = cqs.cqs_plan(out_dtype="f32", **kw)
            ws = torch.empty(cqs.cqs_forward_workspace_size(p)[0], dtype=torch.uint8, device=DEV)
            out = torch.empty(q.shape, dtype=torch.float32, device=DEV)
            lse = torch.empty(q.shape[:3], dtype=torch.float32, device=DEV)
            cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, None)
        torch.cuda.synchronize()
        assert p.info().my_tasks <= len(sub)
        # token-major partial for cqs_merge: [N][B*H][D], [N][B*H]
        res.append((out.to(DEV).permute(2, 0, 1, 3).reshape(N, B * H, D).contiguous(),
                    lse.to(DEV).permute(2, 0, 1).reshape(N, B * H).contiguous()))
    fo = torch.empty(B, H, N, D, dtype=torch.float32, device=DEV)
    fl = torch.empty(B, H, N, dtype=torch.float32, device=DEV)
    cqs.cqs_merge(N, B, H, D, [r[0] for r in res], [r[1] for r in res], out=fo, lse_out=fl)
    torch.cuda.synchronize()
    check_bf16(fo, fl, *ref_dense(q, k, v))


@pytest.mark.parametrize("P,N,depth,D", [(2, 3000, 2, 128), (4, 2401, 3, 64), (8, 5000, 4, 128),
                                         (3, 1030, 2, 64)])
def test_parallel_task_slots(P, N, depth, D):
    """n_parallel = P: tasks round-robin over P streams, each with its own accumulator
    slot, folded together at the end — equals dense attention, and differs from the one-stream
    result only by fp rounding."""
    q, k, v = gen(1, 2, N, D, 700 + P + N, bf16=True)
    res = []
    for n_par in (1, P):
        p = cqs.cqs_plan(N=N, B=1, H=2, D=D, depth=depth, n_parallel=n_par)
        ws = torch.empty(cqs.cqs_forward_workspace_size(p)[0], dtype=torch.uint8, device=DEV)
        out = torch.empty_like(q)
        lse = torch.empty(1, 2, N, dtype=torch.float32, device=DEV)
        st = cqs.cqs_attention_forward(p, q, k, v, out, lse, 0.0, 0, ws, None, stats=True)
        torch.cuda.synchronize()
        assert st.tasks_run == p.info().my_tasks
        res.append((out.clone(), lse.clone()))
    check_bf16(*res[1], *ref_dense(q, k, v))
    assert (res[0][0].float() - res[1][0].float()).abs().max().item() <= 1e-2
    assert (res[0][1] - res[1][1]).abs().max().item() <= 1e-5

"""Pins for oracle O1 (dense attention), O3 (literal Algorithm 1) and O4 (LSE form + merge).

O1 is pinned to: closed forms (N=1 -> O=V; Q=K=0 -> mean of V), an independent
pure-Python loop evaluation with math.exp, and torch's float64 scaled_dot_product_attention (a
library routine).  O3/O4 are pinned to O1 ("exactly the same result as full-sequence attention",
P:8) at several depths, to each other, and by negative controls (dropping a task / a mask group
must break them by far more than the tolerance)."""
import math

import numpy as np
import pytest
import torch

import cqs_synth
from oracle import cqs_oracle as O

I = (0, 1, 3)


def qkv(B, H, N, D, seed=1, scale=1.0):
    return tuple(scale * cqs_synth.numpy_tensor((B, H, N, D), seed, n) for n in ("q", "k", "v"))


def loop_attention(q, k, v):
    """Independent brute force: per row, per key, math.exp — no NumPy vector ops."""
    N, D = len(q), len(q[0])
    a = 1.0 / math.sqrt(D)
    out, lses = [], []
    for i in range(N):
        logits = [a * sum(q[i][d] * k[j][d] for d in range(D)) for j in range(N)]
        mx = max(logits)
        w = [math.exp(x - mx) for x in logits]
        s = sum(w)
        out.append([sum(w[j] * v[j][d] for j in range(N)) / s for d in range(D)])
        lses.append(mx + math.log(s))
    return out, lses


def test_dense_n1_is_v():
    q, k, v = qkv(1, 2, 1, 8)
    Ov, lse = O.dense_attention(q, k, v)
    assert np.array_equal(Ov, v)
    assert np.allclose(lse[..., 0], np.einsum("bhnd,bhnd->bhn", q, k)[..., 0] / math.sqrt(8))


def test_dense_zero_qk_is_mean_v():
    _, _, v = qkv(1, 1, 9, 4)
    z = np.zeros_like(v)
    Ov, lse = O.dense_attention(z, z, v)
    assert np.allclose(Ov, v.mean(axis=2, keepdims=True).repeat(9, axis=2), atol=1e-15)
    assert np.allclose(lse, math.log(9))


def test_dense_matches_loop_form():
    q, k, v = qkv(1, 1, 11, 5, seed=3)
    Ov, lse = O.dense_attention(q, k, v)
    lo, ll = loop_attention(q[0, 0].tolist(), k[0, 0].tolist(), v[0, 0].tolist())
    assert np.allclose(Ov[0, 0], np.array(lo), rtol=0, atol=1e-13)
    assert np.allclose(lse[0, 0], np.array(ll), rtol=0, atol=1e-13)


def test_dense_matches_torch_sdpa_f64():
    q, k, v = qkv(2, 3, 40, 16, seed=5)
    Ov, _ = O.dense_attention(q, k, v)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v)).numpy()
    assert np.allclose(Ov, ref, rtol=0, atol=1e-13)


def test_dense_rows_matches_dense():
    q, k, v = qkv(1, 1, 300, 16, seed=7)
    Ov, lse = O.dense_attention(q, k, v)
    rows = np.array([0, 17, 299, 150])
    o2, l2 = O.dense_attention_rows(q[0, 0], k[0, 0], v[0, 0], rows, block=64)
    assert np.allclose(o2, Ov[0, 0, rows], atol=1e-14) and np.allclose(l2, lse[0, 0, rows], atol=1e-13)


CASES = [(7, 1), (21, 1), (49, 1), (49, 2), (147, 2), (448, 1), (343, 3)]


@pytest.mark.parametrize("N,itr", CASES)
def test_alg1_equals_dense(N, itr):
    q, k, v = qkv(1, 2, N, 8, seed=N + itr)
    ents = O.build_subseq(N, 7, itr, I)
    Od, lse_d = O.dense_attention(q, k, v)
    O1, Den = O.cqsa_forward_alg1(q, k, v, ents)
    assert np.max(np.abs(O1 - Od)) / np.max(np.abs(Od)) < 1e-10
    assert np.allclose(np.log(Den), lse_d, rtol=0, atol=1e-10)


@pytest.mark.parametrize("N,itr", [(21, 1), (49, 2), (343, 3)])
def test_lse_form_equals_alg1_and_dense(N, itr):
    q, k, v = qkv(1, 1, N, 8, seed=2 * N)
    ents = O.build_subseq(N, 7, itr, I)
    Od, lse_d = O.dense_attention(q, k, v)
    O4, lse4 = O.cqsa_forward_lse(q, k, v, ents)
    O3, _ = O.cqsa_forward_alg1(q, k, v, ents)
    assert np.max(np.abs(O4 - Od)) < 1e-12 and np.max(np.abs(O4 - O3)) < 1e-12
    assert np.max(np.abs(lse4 - lse_d)) < 1e-12


def test_fully_masked_rows_give_neg_inf_partials():
    # at itr >= 3 some leaf rows keep no key -> (O_i=0, lse_i=-inf) and are skipped (R8)
    N = 343
    q, k, v = qkv(1, 1, N, 4, seed=9)
    seen = 0
    for e in O.build_subseq(N, 7, 3, I):
        Oi, li = O.task_partial(q, k, v, e)
        dead = ~O.local_mask(e).any(axis=1)
        seen += dead.sum()
        assert np.all(np.isneginf(li[0, 0, dead])) and np.all(Oi[0, 0, dead] == 0)
        assert np.all(np.isfinite(li[0, 0, ~dead]))
    assert seen > 0


def test_granularity_invariance():
    q, k, v = qkv(2, 2, 49, 8, seed=11)
    a = O.cqsa_forward_alg1(q, k, v, O.build_subseq(49, 7, 1, I))[0]
    b = O.cqsa_forward_alg1(q, k, v, O.build_subseq(49, 7, 2, I))[0]
    assert np.max(np.abs(a - b)) < 1e-12


def test_negative_controls():
    q, k, v = qkv(1, 1, 49, 8, seed=13)
    Od, lse_d = O.dense_attention(q, k, v)
    ents = O.build_subseq(49, 7, 1, I)
    O_drop, _ = O.cqsa_forward_lse(q, k, v, ents[:-1] + [ents[-1]] * 0)  # drop a task
    assert np.max(np.abs(O_drop - Od)) > 1e-3
    ents[3].group_runs = ents[3].group_runs[1:]                          # double-count a block
    O_dup, lse_dup = O.cqsa_forward_lse(q, k, v, ents)
    assert np.max(np.abs(lse_dup - lse_d)) > 1e-3


def test_lse_merge_handles_neg_inf():
    o = np.ones((2, 3))
    m, l = O.lse_merge([(o, np.array([0.0, -np.inf])), (2 * o, np.array([-np.inf, -np.inf]))])
    assert np.allclose(m[0], 1.0) and np.all(m[1] == 0) and l[0] == 0 and np.isneginf(l[1])
    m, l = O.lse_merge([(o, np.log([1.0, 3.0])), (3 * o, np.log([3.0, 1.0]))])
    assert np.allclose(m[0], 2.5) and np.allclose(m[1], 1.5) and np.allclose(l, np.log(4.0))

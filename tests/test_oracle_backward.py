"""Pins for oracle O6 (backward): literal Algorithm 2 against the
closed-form dense gradients, both against central finite differences of L = sum(dO * O) on tiny
inputs, plus the trivial cases of SPEC (dO = 0 -> 0; attention is linear in V)."""
import numpy as np
import pytest

import cqs_synth
from oracle import cqs_oracle as O

I = (0, 1, 3)


def qkvd(B, H, N, D, seed):
    return tuple(cqs_synth.numpy_tensor((B, H, N, D), seed, n) for n in ("q", "k", "v")) + (
        cqs_synth.numpy_tensor((B, H, N, D), seed + 1, "q"),)


def test_dense_grads_match_finite_differences():
    q, k, v, dO = qkvd(1, 1, 7, 3, 5)
    loss = lambda q_, k_, v_: float((O.dense_attention(q_, k_, v_)[0] * dO).sum())
    dQ, dK, dV = O.dense_attention_grads(q, k, v, dO)
    h = 1e-6
    for name, x, g in (("q", q, dQ), ("k", k, dK), ("v", v, dV)):
        for idx in [(0, 0, 0, 0), (0, 0, 3, 1), (0, 0, 6, 2), (0, 0, 2, 0)]:
            xp, xm = x.copy(), x.copy()
            xp[idx] += h
            xm[idx] -= h
            args_p = {"q": (xp, k, v), "k": (q, xp, v), "v": (q, k, xp)}[name]
            args_m = {"q": (xm, k, v), "k": (q, xm, v), "v": (q, k, xm)}[name]
            fd = (loss(*args_p) - loss(*args_m)) / (2 * h)
            assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(g[idx])), (name, idx, fd, g[idx])


def test_trivial_cases():
    q, k, v, dO = qkvd(1, 2, 9, 4, 7)
    z = np.zeros_like(dO)
    for g in O.dense_attention_grads(q, k, v, z):
        assert np.all(g == 0)
    # linear in V: dV does not depend on V
    dV1 = O.dense_attention_grads(q, k, v, dO)[2]
    dV2 = O.dense_attention_grads(q, k, 3 * v - 1, dO)[2]
    assert np.allclose(dV1, dV2, atol=1e-14)


@pytest.mark.parametrize("N,itr", [(7, 1), (21, 1), (49, 2), (147, 2), (343, 3)])
def test_alg2_equals_dense_grads(N, itr):
    q, k, v, dO = qkvd(1, 2, N, 8, 11 + N)
    ents = O.build_subseq(N, 7, itr, I)
    ref = O.dense_attention_grads(q, k, v, dO)
    got = O.cqsa_backward_alg2(q, k, v, dO, ents)
    for r, g in zip(ref, got):
        assert np.max(np.abs(g - r)) / np.max(np.abs(r)) < 1e-10


def test_alg2_negative_control():
    q, k, v, dO = qkvd(1, 1, 49, 8, 3)
    ents = O.build_subseq(49, 7, 1, I)
    ents[2].group_runs = ents[2].group_runs[1:]          # double-count a diagonal block
    ref = O.dense_attention_grads(q, k, v, dO)
    got = O.cqsa_backward_alg2(q, k, v, dO, ents)
    assert max(np.max(np.abs(g - r)) for g, r in zip(got, ref)) > 1e-3


def test_dense_dq_rows_matches_full_gradient():
    """The row-streamed dQ (used for sampled rows at full size) equals dense_attention_grads' dQ,
    itself pinned to finite differences above; small blocks force several key blocks."""
    rng = np.random.default_rng(12)
    N, D = 300, 16
    q, k, v, dO = (rng.standard_normal((1, 1, N, D)) for _ in range(4))
    dQ, _, _ = O.dense_attention_grads(q, k, v, dO)
    rows = np.array([0, 7, 150, 299])
    got = O.dense_dq_rows(q[0, 0], k[0, 0], v[0, 0], dO[0, 0], rows, block=64)
    assert np.abs(got - dQ[0, 0, rows]).max() < 1e-12

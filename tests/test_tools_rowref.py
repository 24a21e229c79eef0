"""The measurement tools' sampled-row reference (tools/_rowref.py, used by tools/c3_bench.py and
tools/c5_scaled.py so that they do not import oracle/) agrees with the oracle's dense attention
and dense gradients on small inputs."""
import numpy as np

from oracle import cqs_oracle as O
from tools import _rowref as R


def test_rows_forward_matches_oracle_dense():
    rng = np.random.default_rng(11)
    q, k, v = (rng.standard_normal((257, 32)) for _ in range(3))
    rows = np.array([0, 1, 128, 255, 256])
    o, lse = R.rows_forward(q, k, v, rows, block=50)
    Oref, lref = O.dense_attention(q[None, None], k[None, None], v[None, None])
    assert np.abs(o - Oref[0, 0, rows]).max() < 1e-12
    assert np.abs(lse - lref[0, 0, rows]).max() < 1e-12


def test_rows_dq_matches_oracle_dense_grads():
    rng = np.random.default_rng(12)
    q, k, v, do = (rng.standard_normal((130, 16)) for _ in range(4))
    rows = np.array([0, 64, 129])
    dq = R.rows_dq(q, k, v, do, rows, block=40)
    ref = O.dense_attention_grads(q[None, None], k[None, None], v[None, None], do[None, None])[0]
    assert np.abs(dq - ref[0, 0, rows]).max() < 1e-11

"""Sampled-row references for the scaled measurement tools (c3_bench.py, c5_scaled.py).

fp64 NumPy, keys streamed in blocks: O_r = softmax(alpha q_r K^T) V and lse_r for the sampled query
rows r, and dQ_r of L = sum dO . O.  Written independently of oracle/ (which only tests/, smoke()
and bench.py's cpu_baseline leg use); the parity claims that gate the product are the tests'."""
import math

import numpy as np


def rows_forward(q, k, v, rows, block=1 << 18):
    """O and lse (natural log) of query `rows` of one [N, D] plane: exact max pass, then sums."""
    N, D = k.shape
    a = 1.0 / math.sqrt(D)
    qr = np.asarray(q[rows], np.float64)
    mx = np.full(len(rows), -np.inf)
    for s in range(0, N, block):
        mx = np.maximum(mx, (a * qr @ np.asarray(k[s:s + block], np.float64).T).max(axis=1))
    den = np.zeros(len(rows))
    num = np.zeros((len(rows), v.shape[1]))
    for s in range(0, N, block):
        e = np.exp(a * qr @ np.asarray(k[s:s + block], np.float64).T - mx[:, None])
        den += e.sum(axis=1)
        num += e @ np.asarray(v[s:s + block], np.float64)
    return num / den[:, None], mx + np.log(den)


def rows_dq(q, k, v, dO, rows, block=1 << 18):
    """dQ_r = alpha sum_j P_rj (dO_r . v_j - dO_r . O_r) k_j for query `rows`."""
    N, D = k.shape
    a = 1.0 / math.sqrt(D)
    o, lse = rows_forward(q, k, v, rows, block)
    qr = np.asarray(q[rows], np.float64)
    dor = np.asarray(dO[rows], np.float64)
    delta = (dor * o).sum(axis=1)
    dq = np.zeros((len(rows), D))
    for s in range(0, N, block):
        kb = np.asarray(k[s:s + block], np.float64)
        vb = np.asarray(v[s:s + block], np.float64)
        p = np.exp(a * qr @ kb.T - lse[:, None])
        dq += (p * (dor @ vb.T - delta[:, None])) @ kb
    return a * dq

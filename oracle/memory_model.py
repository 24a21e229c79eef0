"""ORACLE O5 — device-memory model M_dev and budget-driven depth choice.  TEST INFRASTRUCTURE ONLY.

The paper fixes the law, not the bytes: "each CQS Divide reduces the memory footprint by a factor of
l/c = 3/7" for a linear per-task memory Mem(x) = D x + E, and uniform
scheduling picks the divide granularity so that one task fits the memory limit (P:146, P:152,
P:162).  The byte terms below are this build's accounting (reading R14):
everything live on the device during a forward call = caller device tensors + the workspace.

Pins (tests/test_oracle_memory.py): the staging term shrinks by ~3/7 per level, task count
c^k, leaf length N(3/7)^k +- k, monotone feasibility in the budget.
"""
from __future__ import annotations

from oracle import cqs_oracle as O

FLUSH_BYTES = 256 << 20   # two flush buffers of ~FLUSH_BYTES each


def flush_rows(acc_rows, BH, D):
    f = FLUSH_BYTES // (BH * (D + 1) * 4)
    return min(max(f, 1024), 65536, acc_rows)


def _a256(x):
    return (x + 255) // 256 * 256


def _alloc(x):
    """Bytes a separately allocated device tensor occupies (R14): < 1 MiB -> 512-byte multiple
    (shared small segment); otherwise its own segment of 2 MiB device pages."""
    if x < (1 << 20):
        return (x + 511) // 512 * 512
    return (x + (2 << 20) - 1) // (2 << 20) * (2 << 20)


def leaf_staged_rows(N, c, I, k):
    """Largest number of rows any non-empty leaf must stage: segments that are a query or key of a
    kept block.  Uses the literal Alg. 3 entry and its mask groups."""
    best = 0
    for qt in O.quorum_tuples(c, k):
        e = O.build_subseq_entry(N, c, I, qt)
        segs = O.entry_segments(e)
        kept = O.segment_kept_matrix(e, segs)
        used = kept.any(axis=0) | kept.any(axis=1)
        best = max(best, sum(s[1] for s, u in zip(segs, used) if u))
    return best


def node_rows_max(N, c, I, j):
    """Longest depth-j subsequence (P:279-283 layout applied j times)."""
    lens = {N}
    for _ in range(j):
        nxt = set()
        for L in lens:
            st, en = O.balanced_chunk_layout(L, c)
            for q in range(c):
                nxt.add(sum(en[(q + o) % c] - st[(q + o) % c] for o in I))
        lens = nxt
    return max(lens)


def workspace_bytes(N, BH, D, e_in, streamed, out_host, staged_rows, acc_rows, nbuf,
                    n_parallel=1):
    b = _a256(acc_rows * BH * D * 4) + _a256(acc_rows * BH * 4)
    if not streamed and n_parallel > 1:   # accumulator slots of concurrently running tasks
        b += (n_parallel - 1) * (_a256(acc_rows * BH * D * 4) + _a256(acc_rows * BH * 4))
    if streamed:
        b += nbuf * 3 * _a256(BH * staged_rows * D * e_in)
    if streamed or out_host:
        F = flush_rows(acc_rows, BH, D)
        b += 2 * (_a256(F * BH * D * 4) + _a256(F * BH * 4))
    return b


def device_bytes(N, B, H, D, e_in, e_out, streamed, out_host, staged_rows, acc_rows, nbuf,
                 n_parallel=1):
    """Each tensor as the caller's allocator holds it (_alloc, R14)."""
    BH = B * H
    caller = 0 if streamed else 3 * _alloc(BH * N * D * e_in)
    if not out_host:
        caller += _alloc(BH * N * D * e_out) + _alloc(4 * BH * N)
    return caller + _alloc(workspace_bytes(N, BH, D, e_in, streamed, out_host, staged_rows,
                                          acc_rows, nbuf, n_parallel))


def choose(N, B, H, D, e_in, e_out, streamed, out_host, budget, c=7, I=(0, 1, 3), depth=None,
           staged=None):
    """Smallest depth k (then nbuf 2 before 1, then smallest accumulator depth j) whose predicted
    device bytes fit the budget (uniform scheduling).  Returns (k, j, nbuf, bytes) or None.
    `staged` may pass precomputed leaf_staged_rows per k (they are expensive for big N)."""
    kmax = 0
    while c ** (kmax + 1) <= N and kmax + 1 < 12:
        kmax += 1
    ks = [depth] if depth is not None else range(0, kmax + 1)
    for k in ks:
        if not streamed:
            b = device_bytes(N, B, H, D, e_in, e_out, False, out_host, 0, N, 0)
            if budget == 0 or b <= budget:
                return k, 0, 0, b
            continue
        Lh = staged[k] if staged is not None else leaf_staged_rows(N, c, I, k)
        for nbuf in (2, 1):
            for j in range(0, k + 1):
                b = device_bytes(N, B, H, D, e_in, e_out, True, out_host, Lh,
                                 node_rows_max(N, c, I, j), nbuf)
                if budget == 0 or b <= budget:
                    return k, j, nbuf, b
    return None


# ---- backward (Algorithm 2, NEXT-1) device workspace: this build's accounting (DESIGN.md
#      "Backward kernels"); the paper only reports Mem_bwd ~ 2 x Mem_fwd ----

def backward_workspace_bytes(N, BH, D, streamed=False, staged_rows=0, nbuf=0):
    """lse/Delta table [BH][2][ceil4(N)] fp32 + three fp32 gradient accumulators [N][BH][D];
    streamed adds nbuf staging buffers of four bf16 tensors [BH][staged_rows][D] and two chunk
    buffers of F rows (F = clamp(64 MiB / (BH D 4), 256, 65536), at most N) holding F x BH x D
    fp32 + F x BH fp32 each."""
    pitch = (N + 3) // 4 * 4
    b = _a256(BH * 2 * pitch * 4) + 3 * _a256(N * BH * D * 4)
    if streamed:
        b += nbuf * 4 * _a256(BH * staged_rows * D * 2)
        F = min(max((64 << 20) // (BH * D * 4), 256), 65536, N)
        b += 2 * (_a256(F * BH * D * 4) + _a256(F * BH * 4))
    return _alloc(b)

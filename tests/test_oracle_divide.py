"""Pins for oracle O2: literal Algorithm 3 BuildSubseq, the CQS mask
and the canonical segment form.  Pins come from the paper's printed facts (Eq. 1, Fig. 2, Fig. 3,
Sec. 2.3) and brute-force pair coverage ("covered exactly once")."""
import numpy as np
import pytest

from conftest import read_golden
from oracle import cqs_oracle as O

I = (0, 1, 3)


def _golden_kv(name):
    out = {}
    for ln in read_golden(name):
        k, v = ln.split(":", 1)
        out[k.strip()] = v.strip()
    return out


def test_eq1_n7():
    ents = O.build_subseq(7, 7, 1, I)
    gold = {int(k): list(map(int, v.split())) for k, v in _golden_kv("eq1_n7_itr1.txt").items()}
    assert [e.quorum for e in ents] == [(i,) for i in range(7)]
    for i, e in enumerate(ents):
        assert e.token_ids.tolist() == gold[i]


def test_fig2_diagonal_pair_ownership():
    ln = read_golden("fig2_diag_pairs.txt")[0]
    chunk, rest = ln.split(":")
    holders, keeper = rest.split(";")
    chunk, holders, keeper = int(chunk), list(map(int, holders.split())), int(keeper)
    ents = O.build_subseq(7, 7, 1, I)
    assert [i for i, e in enumerate(ents) if chunk in e.token_ids.tolist()] == holders
    for i in holders:                     # token `chunk` attends itself only in the keeper
        e = ents[i]
        p = e.token_ids.tolist().index(chunk)
        assert O.local_mask(e)[p, p] == (1.0 if i == keeper else 0.0)


def test_seq0_masks_11_and_33():
    # Seq_0 holds (0,0),(1,1),(3,3); only (0,0) retained.  N=21 -> chunks of 3 tokens.
    e = O.build_subseq(21, 7, 1, I)[0]
    M = O.local_mask(e)
    assert M[0:3, 0:3].all() and not M[3:6, 3:6].any() and not M[6:9, 6:9].any()
    assert M[0:3, 3:9].all() and M[3:6, 6:9].all()   # off-diagonal chunk pairs kept


def test_fig3_n49():
    g = _golden_kv("fig3_n49.txt")
    e1 = O.build_subseq(49, 7, 1, I)
    assert len(e1) == int(g["itr1_n_entries"])
    assert all(len(e.token_ids) == int(g["itr1_len"]) for e in e1)
    assert e1[0].token_ids.tolist() == list(map(int, g["itr1_entry0_tokens"].split()))
    M = O.local_mask(e1[0])
    blocks = [tuple(map(int, b.split())) for b in g["itr1_entry0_masked_blocks"].split(";")]
    Z = np.ones_like(M)
    for s, t in blocks:
        Z[s:t, s:t] = 0
    assert np.array_equal(M, Z)
    e2 = O.build_subseq(49, 7, 2, I)
    assert len(e2) == int(g["itr2_n_entries"])
    assert all(len(e.token_ids) == int(g["itr2_len"]) for e in e2)
    s2, _ = O.balanced_chunk_layout(21, 7)
    assert s2[1] - s2[0] == int(g["itr2_chunk"])
    # itr=2 entries carry local AND inherited masks: more than (l-1) masked groups
    assert any(len(e.group_runs) > 2 for e in e2)


def test_balanced_layout():
    assert O.balanced_chunk_layout(49, 7) == (list(range(0, 49, 7)), list(range(7, 50, 7)))
    st, en = O.balanced_chunk_layout(10, 7)
    assert [b - a for a, b in zip(st, en)] == [2, 2, 2, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        O.balanced_chunk_layout(5, 7)


def test_indices_to_runs():
    assert O.indices_to_runs([3, 4, 5, 9]) == [(3, 6), (9, 10)]
    assert O.indices_to_runs([]) == []
    assert O.indices_to_runs([0]) == [(0, 1)]


CASES = [(N, itr) for itr in (1, 2) for N in (7 ** itr, 7 ** itr + 5, 3 * 7 ** itr + 1)] + \
        [(343, 3), (348, 3)]


@pytest.mark.parametrize("N,itr", CASES)
def test_coverage_exactly_once(N, itr):
    """Every ordered token pair is kept in exactly one task (P:83 'covered exactly once')."""
    ents = O.build_subseq(N, 7, itr, I)
    cnt = O.coverage_counts(ents, N)
    assert cnt.min() == 1 and cnt.max() == 1


@pytest.mark.parametrize("N,itr", [(20, 1), (60, 2)])
def test_coverage_paired_set(N, itr):
    ents = O.build_subseq(N, 7, itr, (0, 1, 5))
    cnt = O.coverage_counts(ents, N)
    assert cnt.min() == 1 and cnt.max() == 1


def test_coverage_c13():
    # Appendix B figure: full coverage for c=13, I=(0,1,3,9)
    ents = O.build_subseq(169, 13, 1, (0, 1, 3, 9))
    cnt = O.coverage_counts(ents, 169)
    assert cnt.min() == 1 and cnt.max() == 1


def test_negative_control_dropped_group():
    ents = O.build_subseq(49, 7, 1, I)
    ents[2].group_runs = ents[2].group_runs[1:]
    cnt = O.coverage_counts(ents, 49)
    assert cnt.max() == 2


@pytest.mark.parametrize("N,itr", [(49, 2), (100, 2), (400, 3)])
def test_counts_multiplicity_lengths(N, itr):
    ents = O.build_subseq(N, 7, itr, I)
    assert len(ents) == 7 ** itr                                  # n_total = c^itr
    occ = np.zeros(N, dtype=int)
    for e in ents:
        occ[e.token_ids] += 1
        assert len(np.unique(e.token_ids)) == len(e.token_ids)
        assert abs(len(e.token_ids) - N * (3 / 7) ** itr) <= itr  # lengths ~ N (l/c)^itr
    assert (occ == 3 ** itr).all()                                # each chunk in l subsequences


@pytest.mark.parametrize("itr", [1, 2, 3])
def test_kept_area(itr):
    N = 7 ** itr
    ents = O.build_subseq(N, 7, itr, I)
    kept = [O.local_mask(e).sum() for e in ents]
    assert sum(kept) == N * N
    L = len(ents[0].token_ids)
    assert np.isclose(np.mean(kept) / L ** 2, (7 / 9) ** itr)


@pytest.mark.parametrize("N,itr", [(49, 1), (49, 2), (54, 2), (348, 3)])
def test_segments_reproduce_mask(N, itr):
    """The canonical segment form is lossless: expanding segment kept-blocks gives the literal M_i,
    and segments tile token_ids in order."""
    for e in O.build_subseq(N, 7, itr, I):
        segs = O.entry_segments(e)
        kept = O.segment_kept_matrix(e, segs)
        ids = np.concatenate([np.arange(s, s + ln) for s, ln, _ in segs])
        assert np.array_equal(ids, e.token_ids)
        lens = [ln for _, ln, _ in segs]
        M = np.kron(np.ones((1, 1)), np.block([[np.full((lens[a], lens[b]), float(kept[a, b]))
                                                for b in range(len(segs))] for a in range(len(segs))]))
        assert np.array_equal(M, O.local_mask(e))
        assert O.entry_work(segs, kept) == O.local_mask(e).sum()


def test_empty_tasks_at_depth3():
    # at itr=3, 7 of 343 leaves keep no pair at all
    ents = O.build_subseq(343, 7, 3, I)
    empty = [e.quorum for e in ents if O.local_mask(e).sum() == 0]
    assert len(empty) == 7 and all(q[1] == 5 and q[2] == 0 for q in empty)


def test_plan_bytes_deterministic_header():
    b = O.plan_bytes(49, 7, I, 1)
    assert b[:4] == b"CQSP" and O.plan_bytes(49, 7, I, 1) == b

"""GPU-free parity of the C++ planner (cqs_plan) against the oracle's literal Algorithm 3
(PAPER.md P:269-307): canonical plan bytes must be bit-identical ("bit-exact for the plan
and task lists")."""
import numpy as np
import pytest

import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O

I = (0, 1, 3)


def _plan(N, depth, **kw):
    return cqs.cqs_plan(N=N, B=1, H=1, D=64, depth=depth, in_dtype="f32", **kw)


CASES = [(7, 1), (10, 1), (49, 1), (448, 1), (49, 2), (54, 2), (100, 2), (343, 3), (348, 3),
         (1030, 3), (2401, 4), (3000, 4), (131072, 1), (7 ** 5, 5)]


@pytest.mark.parametrize("N,itr", CASES)
def test_plan_bytes_bit_exact(N, itr):
    assert cqs.cqs_plan_serialize(_plan(N, itr)) == O.plan_bytes(N, 7, I, itr)


@pytest.mark.parametrize("N,itr", [(60, 2), (400, 3)])
def test_plan_bytes_paired_set(N, itr):
    p = cqs.cqs_plan(N=N, B=1, H=1, D=64, depth=itr, in_dtype="f32", offsets=(0, 1, 5))
    assert cqs.cqs_plan_serialize(p) == O.plan_bytes(N, 7, (0, 1, 5), itr)


def test_plan_bytes_c13():
    p = cqs.cqs_plan(N=200, B=1, H=1, D=64, depth=1, in_dtype="f32", c=13, offsets=(0, 1, 3, 9))
    assert cqs.cqs_plan_serialize(p) == O.plan_bytes(200, 13, (0, 1, 3, 9), 1)


@pytest.mark.parametrize("N,itr,sample", [(1_000_000, 2, 12), (16_777_216, 3, 6)])
def test_plan_tasks_sampled_large(N, itr, sample):
    """BASELINE configs 2/3 sizes: compare sampled tasks with the literal per-task Alg. 3."""
    p = _plan(N, itr)
    info = p.info()
    assert info.n_tasks == 7 ** itr and info.total_work_pairs == N * N
    rng = np.random.default_rng(0)
    for idx in sorted(rng.choice(7 ** itr, size=sample, replace=False)):
        t = p.task(int(idx))
        qt = tuple(int(t.quorum[i]) for i in range(itr))
        e = O.build_subseq_entry(N, 7, I, qt)
        segs = O.entry_segments(e)
        kept = O.segment_kept_matrix(e, segs)
        assert t.nseg == len(segs)
        for a, (st, ln, cd) in enumerate(segs):
            assert (t.seg_start[a], t.seg_len[a]) == (st, ln)
            assert tuple(t.seg_codes[a][:itr]) == cd
            assert t.kept[a] == sum(1 << b for b in range(len(segs)) if kept[a, b])
        assert t.work == O.entry_work(segs, kept)


def test_plan_info_counts():
    info = _plan(343, 3).info()
    assert info.n_tasks == 343 and info.n_empty == 7 and info.total_work_pairs == 343 ** 2


@pytest.mark.parametrize("world", [2, 3, 8])
def test_lpt_sharding_covers_tasks_once(world):
    N, itr = 2401, 4
    plans = [cqs.cqs_plan(N=N, B=1, H=1, D=64, depth=itr, in_dtype="f32", world=world, rank=r)
             for r in range(world)]
    infos = [p.info() for p in plans]
    assert sum(i.my_work_pairs for i in infos) == N * N
    assert sum(i.my_tasks for i in infos) == 7 ** itr - infos[0].n_empty
    ranks = [plans[0].task(i).rank for i in range(7 ** itr)]
    for i in range(0, 7 ** itr, 97):                       # every rank sees the same assignment
        assert all(p.task(i).rank == ranks[i] for p in plans)
    loads = [i.my_work_pairs for i in infos]
    assert max(loads) / (sum(loads) / world) < 1.05         # LPT balance at depth 4


def test_plan_deterministic():
    a = cqs.cqs_plan_serialize(_plan(1030, 3))
    b = cqs.cqs_plan_serialize(_plan(1030, 3))
    assert a == b


@pytest.mark.parametrize("c,I,N,itr", [(13, (0, 1, 3, 9), 400, 2), (21, (0, 1, 4, 14, 16), 500, 1),
                                       (13, (0, 1, 5, 11), 300, 1)])
def test_plan_bytes_other_interest_sets(c, I, N, itr):
    """NEXT-3: larger cyclic difference sets (Appendix B table, and the
    paired set of (0,1,3,9)) plan bit-exactly like c=7."""
    p = cqs.cqs_plan(N=N, B=1, H=1, D=64, depth=itr, in_dtype="f32", c=c, offsets=I)
    assert cqs.cqs_plan_serialize(p) == O.plan_bytes(N, c, I, itr)
    assert p.info().total_work_pairs == N * N

"""Hybrid scheduling (NEXT-2, Fig. "schedule" right; DESIGN reading R20):
leaves at mixed depths.  The C++ planner's hybrid tree must equal the oracle's rule leaf for leaf
(bit-exact canonical bytes), be a complete c-ary tree (so every ordered pair is covered exactly
once), reproduce dense attention through the oracle, and balance the LPT makespan."""
import numpy as np
import pytest

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O

I = (0, 1, 3)


def hybrid(N, world, depth=1, rank=0):
    return cqs.cqs_plan(N=N, B=1, H=1, D=64, depth=depth, in_dtype="bf16", world=world, rank=rank,
                        schedule="hybrid")


def leaves_of(p):
    out = []
    for t in range(p.info().n_tasks):
        T = p.task(t)
        out.append(tuple(int(T.quorum[i]) for i in range(T.depth)))
    return out


@pytest.mark.parametrize("N,world,depth", [(500, 2, 1), (3000, 8, 1), (3000, 3, 1), (4000, 4, 2),
                                           (131072, 8, 1)])
def test_hybrid_tree_matches_oracle_rule(N, world, depth):
    p = hybrid(N, world, depth)
    got = leaves_of(p)
    assert got == O.hybrid_leaves(N, 7, I, depth, world)
    info = p.info()
    assert info.depth == depth and info.max_depth == max(len(q) for q in got)
    if N <= 4000:
        assert cqs.cqs_plan_serialize(p) == O.hybrid_plan_bytes(N, 7, I, depth, got)


@pytest.mark.parametrize("N,world", [(3000, 8), (131072, 8), (131072, 3), (1_000_000, 8)])
def test_hybrid_is_complete_tree_and_balanced(N, world):
    p = hybrid(N, world)
    info = p.info()
    leaves = leaves_of(p)
    # complete prefix code: Kraft sum exactly 1 and no leaf is a prefix of another
    from fractions import Fraction
    assert sum(Fraction(1, 7 ** len(q)) for q in leaves) == 1
    ls = set(leaves)
    for q in leaves:
        for j in range(len(q)):
            assert q[:j] not in ls
    assert info.total_work_pairs == N * N
    loads = [0] * world
    for t in range(info.n_tasks):
        T = p.task(t)
        if T.work:
            loads[T.rank] += T.work
    assert max(loads) <= 1.01 * N * N / world
    # every rank plans the same tree
    assert leaves_of(hybrid(N, world, rank=world - 1)) == leaves


def test_hybrid_covers_every_pair_exactly_once():
    """Brute force (Fig. 2 "covered exactly once") on a mixed-depth tree."""
    N = 300
    leaves = O.hybrid_leaves(N, 7, I, 1, 8)
    assert len({len(q) for q in leaves}) > 1
    ents = [O.build_subseq_entry(N, 7, I, q) for q in leaves]
    assert (O.coverage_counts(ents, N) == 1).all()


def test_hybrid_reproduces_dense_attention():
    N, H, D = 300, 2, 16
    leaves = O.hybrid_leaves(N, 7, I, 1, 8)
    ents = [O.build_subseq_entry(N, 7, I, q) for q in leaves]
    q, k, v = (cqs_synth.numpy_tensor((1, H, N, D), 5, n) for n in ("q", "k", "v"))
    Oh, lh = O.cqsa_forward_lse(q, k, v, ents)
    Od, ld = O.dense_attention(q, k, v)
    assert np.abs(Oh - Od).max() < 1e-12 and np.abs(lh - ld).max() < 1e-12


def test_hybrid_world1_is_uniform_and_streamed_rejected():
    a = cqs.cqs_plan_serialize(hybrid(3000, 1))
    b = cqs.cqs_plan_serialize(cqs.cqs_plan(N=3000, B=1, H=1, D=64, depth=1, in_dtype="bf16"))
    assert a == b
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=3000, B=1, H=1, D=64, depth=1, in_dtype="bf16", qkv_loc="host",
                     world=2, schedule="hybrid")
    assert e.value.status == cqs.CQS_E_UNSUPPORTED

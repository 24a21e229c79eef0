"""Per-level interest sets (NEXT-3; "different values of c can be used at each
iteration"; DESIGN reading R21): the C++ planner's mixed-c tree must be bit-identical to the literal
per-level Algorithm 3 of the oracle, cover every ordered pair exactly once, and reproduce dense
attention through the oracle."""
import numpy as np
import pytest

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O

S7, S7P, S13, S21 = (7, (0, 1, 3)), (7, (0, 1, 5)), (13, (0, 1, 3, 9)), (21, (0, 1, 4, 14, 16))
CASES = [(500, [S7, S13], 2), (500, [S13, S7], 2), (300, [S7, S7P], 2), (1200, [S21, S7], 2),
         (2000, [S7, S13, S7], 3)]


def plan(N, levels, depth, **kw):
    return cqs.cqs_plan(N=N, B=1, H=1, D=64, depth=depth, in_dtype="f32", levels=levels, **kw)


@pytest.mark.parametrize("N,levels,depth", CASES)
def test_mixed_levels_plan_bytes_bit_exact(N, levels, depth):
    p = plan(N, levels, depth)
    info = p.info()
    assert info.n_tasks == int(np.prod([c for c, _ in levels[:depth]]))
    assert info.total_work_pairs == N * N
    assert cqs.cqs_plan_serialize(p) == O.plan_bytes_levels(N, levels, depth)


@pytest.mark.parametrize("N,levels,depth", [(120, [S7, S13], 2), (150, [S13, S7], 2),
                                            (200, [S7, S7P], 2)])
def test_mixed_levels_cover_every_pair_once(N, levels, depth):
    ents = [O.build_subseq_entry_levels(N, levels, qt)
            for qt in O.quorum_tuples_levels([c for c, _ in levels[:depth]])]
    assert (O.coverage_counts(ents, N) == 1).all()


def test_mixed_levels_negative_control():
    """Dropping one leaf of a mixed tree leaves uncovered pairs (the pin can fail)."""
    N, levels = 150, [S13, S7]
    qts = O.quorum_tuples_levels([13, 7])
    ents = [O.build_subseq_entry_levels(N, levels, qt) for qt in qts[:-1]]
    assert (O.coverage_counts(ents, N) == 0).any()


def test_mixed_levels_reproduce_dense_attention():
    N, H, D = 260, 2, 16
    levels = [S13, S7]
    ents = [O.build_subseq_entry_levels(N, levels, qt) for qt in O.quorum_tuples_levels([13, 7])]
    q, k, v = (cqs_synth.numpy_tensor((1, H, N, D), 9, n) for n in ("q", "k", "v"))
    Om, lm = O.cqsa_forward_lse(q, k, v, ents)
    Od, ld = O.dense_attention(q, k, v)
    assert np.abs(Om - Od).max() < 1e-12 and np.abs(lm - ld).max() < 1e-12


def test_levels_beyond_spec_use_base_set_and_validation():
    # one level given, depth 2: level 1 falls back to (c, offsets)
    p = plan(500, [S13], 2)
    assert cqs.cqs_plan_serialize(p) == O.plan_bytes_levels(500, [S13, S7], 2)
    with pytest.raises(cqs.CqsError) as e:
        plan(500, [(7, (0, 1, 2))], 1)
    assert e.value.status == cqs.CQS_E_INVALID
    with pytest.raises(cqs.CqsError) as e:
        plan(500, [(8, (0, 1, 3))], 1)
    assert e.value.status == cqs.CQS_E_INVALID

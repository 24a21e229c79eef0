"""Pins for oracle O0 (interest sets / difference sets), Appendix B."""
import pytest

from conftest import read_golden
from oracle import cqs_oracle as O


def _table():
    rows = []
    for ln in read_golden("interest_sets.txt"):
        head, offs = ln.split(":")
        c, l = map(int, head.split())
        offs = None if offs.strip() == "None" else tuple(map(int, offs.split()))
        rows.append((c, l, offs))
    return rows


def test_chunk_counts_follow_pair_identity():
    # valid c follow {1, 3, 7, 13, 21, ...} for l = 1, 2, 3, 4, 5
    assert [O.chunk_count_for(l) for l in range(1, 6)] == [1, 3, 7, 13, 21]
    for c, l, _ in _table():
        assert O.chunk_count_for(l) == c


def test_base_pattern_is_difference_set():
    assert O.is_difference_set((0, 1, 3), 7)
    assert not O.is_difference_set((0, 1, 2), 7)       # difference 1 appears twice
    assert O.is_difference_set((0,), 1)


def test_c7_prefix01_sets_are_exactly_the_pair():
    # brute force over all 5 candidates (0,1,a): only (0,1,3) and its pair (0,1,5)
    assert O.interest_sets_with_prefix01(7, 3) == [(0, 1, 3), (0, 1, 5)]
    assert O.paired_interest_set((0, 1, 3), 7) == (0, 1, 5)


def test_c13_search_finds_table_set():
    assert (0, 1, 3, 9) in O.interest_sets_with_prefix01(13, 4)


@pytest.mark.parametrize("row", range(10))
def test_table_rows(row):
    c, l, offs = _table()[row]
    if offs is None:
        return
    if l == 12:
        # The printed l=12 set is not a (133,12,1) difference set (R18):
        assert not O.is_difference_set(offs, c)
        assert len(set(O.difference_multiset(offs, c))) < c - 1
        return
    assert O.is_difference_set(offs, c)
    assert O.is_difference_set(tuple(sorted(O.paired_interest_set(offs, c))), c)


def test_cyclic_shift_closure():
    # a difference set stays one under any cyclic shift (differences are shift invariant)
    for s in range(7):
        assert O.is_difference_set(tuple(sorted((a + s) % 7 for a in (0, 1, 3))), 7)
    # a wrong element is detected: (0,1,4) has differences 1,3,4,6,3,... (3 twice)
    assert not O.is_difference_set((0, 1, 4), 7)


def test_difference_set_rejects_bad_input():
    with pytest.raises(ValueError):
        O.is_difference_set((0, 0, 3), 7)
    with pytest.raises(ValueError):
        O.is_difference_set((0, 1, 7), 7)

"""The C-ABI library loads on a CPU-only host and exports every symbol include/cqs.h declares;
host-only entry points (planning, memory model, sharding, error reporting) work without a GPU."""
import ctypes
import os
import re

import pytest

import paper_2604_20819_b200 as cqs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "cqs.h")).read()
    declared = set(re.findall(r"\b(cqs_[a-z_]+)\s*\(", hdr))
    assert declared == set(cqs.ABI_SYMBOLS)
    L = ctypes.CDLL(cqs.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert cqs.lib().cqs_abi_version() == 3


def test_struct_sizes_match_c_layout():
    assert ctypes.sizeof(cqs.PlanDesc) == 104
    assert ctypes.sizeof(cqs.PlanInfo) == 96


def test_invalid_interest_set_rejected():
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=49, B=1, H=1, D=64, depth=1, offsets=(0, 1, 2))
    assert e.value.status == cqs.CQS_E_INVALID and "difference set" in str(e.value)


def test_n_below_c_pow_depth_rejected():
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=48, B=1, H=1, D=64, depth=2)
    assert e.value.status == cqs.CQS_E_INVALID


def test_unsupported_head_dim():
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=49, B=1, H=1, D=96, depth=1, in_dtype="bf16")
    assert e.value.status == cqs.CQS_E_UNSUPPORTED


def test_shard_rows_partition():
    for N, R in [(131072, 8), (1000, 3), (7, 8)]:
        spans = [cqs.cqs_shard_rows(N, R, r) for r in range(R)]
        assert spans[0][0] == 0 and sum(n for _, n in spans) == N
        for (a, n), (b, _) in zip(spans, spans[1:]):
            assert a + n == b


def test_budget_infeasible():
    # resident C2 needs ~6.4 GB: a 1 GiB budget cannot fit at any depth
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=131072, B=1, H=32, D=128, depth=-1, budget_bytes=1 << 30)
    assert e.value.status == cqs.CQS_E_INFEASIBLE

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
    assert cqs.lib().cqs_abi_version() == 5


def test_struct_sizes_match_c_layout(tmp_path):
    """Size and every field offset of the ctypes mirrors equal the C compiler's for include/cqs.h."""
    import os
    import subprocess
    structs = {"cqs_plan_desc": cqs.PlanDesc, "cqs_plan_info_t": cqs.PlanInfo,
               "cqs_task_t": cqs.Task, "cqs_stats": cqs.Stats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cqs.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append('printf("%s %%zu\\n", sizeof(%s));' % (cname, cname))
        for f in py._fields_:
            lines.append('printf("%s.%s %%zu\\n", offsetof(%s, %s));' % (cname, f[0], cname, f[0]))
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                     check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f in py._fields_:
            assert int(got[cname + "." + f[0]]) == getattr(py, f[0]).offset, (cname, f[0])


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


def test_exec_order_must_be_a_permutation():
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=1, exec_order=[0, 1, 2, 3, 4, 5, 5])
    assert e.value.status == cqs.CQS_E_INVALID
    with pytest.raises(cqs.CqsError) as e:
        cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=1, exec_order=[0, 1, 2])
    assert e.value.status == cqs.CQS_E_INVALID
    p = cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=1, exec_order=[6, 5, 4, 3, 2, 1, 0])
    assert p.info().my_tasks == 7


def test_subset_plan_runs_only_listed_tasks():
    p = cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=2, exec_order=[40, 3, 17], subset=True)
    assert p.info().my_tasks == 3 and p.info().n_tasks == 49
    w = sum(p.task(t).work for t in (40, 3, 17))
    assert p.info().my_work_pairs == w
    with pytest.raises(cqs.CqsError):
        cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=2, exec_order=[40, 40], subset=True)


def test_exchange_merge_argument_errors():
    """cqs_exchange_merge rejects world-1 plans and NULL parts before touching the device."""
    import ctypes
    p = cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=1)
    P = ctypes.c_void_p
    st = cqs.lib().cqs_exchange_merge(p.handle, (P * 1)(), (P * 1)(), (ctypes.c_int64 * 1)(), None,
                                      None, None, None)
    assert st == cqs.CQS_E_INVALID
    p2 = cqs.cqs_plan(N=500, B=1, H=1, D=128, depth=1, world=2, rank=0)
    strides = (ctypes.c_int64 * 4)(500 * 128, 500 * 128, 128, 1)
    st = cqs.lib().cqs_exchange_merge(p2.handle, (P * 2)(None, None), (P * 2)(None, None),
                                      (ctypes.c_int64 * 2)(0, 0), P(1 << 20), strides, None, None)
    assert st == cqs.CQS_E_INVALID and b"NULL" in cqs.lib().cqs_last_error()


def test_partial_runs_identity_at_world_one():
    p = cqs.cqs_plan(N=1000, B=1, H=1, D=128, depth=2)
    assert cqs.cqs_partial_runs(p, 0, 100, 50) == [(100, 50, 100)]
    with pytest.raises(cqs.CqsError):
        cqs.cqs_partial_runs(p, 1, 0, 10)

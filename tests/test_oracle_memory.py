"""Pins for oracle O5 (memory model) and its parity with the C++ planner's model.

Paper pins: each divide shrinks the per-task footprint by l/c = 3/7; c^k tasks;
leaf lengths N (3/7)^k."""
import pytest

import paper_2604_20819_b200 as cqs
from oracle import memory_model as M
from oracle import cqs_oracle as O

I = (0, 1, 3)


@pytest.mark.parametrize("N", [7 ** 4, 20000, 100003])
def test_staging_shrinks_by_3_over_7(N):
    prev = None
    for k in range(0, 4):
        Lh = M.leaf_staged_rows(N, 7, I, k)
        assert abs(Lh - N * (3 / 7) ** k) <= k + 1           # ~ N (3/7)^k
        if prev is not None:
            assert abs(Lh / prev - 3 / 7) < 0.01                # factor l/c per divide
        prev = Lh


def test_node_rows():
    assert M.node_rows_max(49, 7, I, 1) == 21 and M.node_rows_max(49, 7, I, 2) == 9
    assert M.node_rows_max(1_000_000, 7, I, 1) == 428572


def _desc(N, B, H, D, streamed, budget, depth=-1):
    return cqs.make_desc(N=N, B=B, H=H, D=D, depth=depth, budget_bytes=budget, in_dtype="bf16",
                         qkv_loc="host" if streamed else "device")


@pytest.mark.parametrize("N,H,D,k,j,nbuf", [(20000, 4, 128, 2, 1, 2), (20000, 4, 64, 1, 0, 1),
                                           (5000, 2, 128, 3, 2, 1)])
def test_cpp_memory_model_matches_oracle(N, H, D, k, j, nbuf):
    d = _desc(N, 1, H, D, True, 0)
    dev, host = cqs.cqs_memory_model(d, k, j, nbuf)
    ref = M.device_bytes(N, 1, H, D, 2, 2, True, True, M.leaf_staged_rows(N, 7, I, k),
                         M.node_rows_max(N, 7, I, j), nbuf)
    assert dev == ref


def test_cpp_depth_choice_matches_oracle():
    N, H, D = 30000, 8, 128
    staged = {k: M.leaf_staged_rows(N, 7, I, k) for k in range(0, 6)}
    for budget in (60_000_000, 80_000_000, 120_000_000, 200_000_000, 10 ** 10):
        ref = M.choose(N, 1, H, D, 2, 2, True, True, budget, staged=staged)
        try:
            info = cqs.cqs_plan(_desc(N, 1, H, D, True, budget)).info()
            got = (info.depth, info.acc_depth, info.n_stage_buffers, info.predicted_peak_bytes)
        except cqs.CqsError as e:
            assert e.status == cqs.CQS_E_INFEASIBLE
            got = None
        assert got == ref, budget


def test_c3_budget_selects_depth_2():
    """BASELINE config 2: N=1M, H=32, D=128, bf16, QKV in pinned host, 16 GiB budget -> depth 2."""
    info = cqs.cqs_plan(_desc(1_000_000, 1, 32, 128, True, 16 << 30)).info()
    assert info.depth == 2 and info.predicted_peak_bytes <= 16 << 30
    staged = {k: M.leaf_staged_rows(1_000_000, 7, I, k) if k < 2 else None for k in range(3)}
    staged[2] = info.max_staged_rows
    ref = M.choose(1_000_000, 1, 32, 128, 2, 2, True, True, 16 << 30, staged=staged)
    assert ref == (info.depth, info.acc_depth, info.n_stage_buffers, info.predicted_peak_bytes)


def test_resident_c2_bytes():
    info = cqs.cqs_plan(_desc(131072, 1, 32, 128, False, 0, depth=1)).info()
    assert info.predicted_peak_bytes == M.device_bytes(131072, 1, 32, 128, 2, 2, False, False, 0,
                                                       131072, 0)


@pytest.mark.parametrize("N,B,H,D", [(131072, 1, 32, 128), (1030, 2, 3, 64), (14458261, 1, 1, 64)])
def test_backward_workspace_matches_c_abi(N, B, H, D):
    """cqs_backward_workspace_size (resident) equals the oracle's byte model; and the streamed
    figure equals it with the plan's staged rows and the staging-buffer count the budget allows."""
    import paper_2604_20819_b200 as cqs
    from oracle import memory_model as M
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=1, in_dtype="bf16")
    assert cqs.cqs_backward_workspace_size(p) == M.backward_workspace_bytes(N, B * H, D)
    ps = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=1, in_dtype="bf16", qkv_loc="host",
                      out_loc="host")
    Lh = ps.info().max_staged_rows
    two = M.backward_workspace_bytes(N, B * H, D, True, Lh, 2)
    assert cqs.cqs_backward_workspace_size(ps) == two
    one = M.backward_workspace_bytes(N, B * H, D, True, Lh, 1)
    assert one < two
    if N == 14458261:   # the C5 scaled backward under 16 GiB takes one staging buffer (14.43 GB)
        assert one <= 16 << 30 < two


@pytest.mark.parametrize("P", [2, 3, 8])
def test_parallel_slots_bytes(P):
    """n_parallel > 1 (resident): one extra fp32 accumulator per additional task in flight."""
    N, B, H, D = 50000, 1, 4, 128
    p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=2, n_parallel=P)
    assert p.info().predicted_peak_bytes == M.device_bytes(N, B, H, D, 2, 2, False, False, 0, N,
                                                          0, n_parallel=P)

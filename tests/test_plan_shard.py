"""Task sharding across ranks and the rank-local accumulator layout
(held row blocks), host logic only."""
import pytest

import paper_2604_20819_b200 as cqs


@pytest.mark.parametrize("shard", ["lpt", "contiguous"])
@pytest.mark.parametrize("N,depth,world", [(2401, 3, 2), (20000, 3, 5), (1 << 24, 3, 8)])
def test_every_task_once_and_rows_held(N, depth, world, shard):
    plans = [cqs.cqs_plan(N=N, B=1, H=8, D=128, depth=depth, world=world, rank=r, shard=shard)
             for r in range(world)]
    info = plans[0].info()
    owner = [plans[0].task(t).rank for t in range(info.n_tasks)]
    assert sum(p.info().my_work_pairs for p in plans) == N * N
    assert sum(p.info().my_tasks for p in plans) == info.n_tasks - info.n_empty
    for t in range(info.n_tasks):
        T = plans[0].task(t)
        assert (T.rank == -1) == (T.work == 0)
        # every active query segment of the task lies in rows its rank holds
        runs = cqs.cqs_partial_runs(plans[0], T.rank, 0, N) if T.rank >= 0 else []
        for a in range(T.nseg):
            if T.kept[a]:
                s, n = T.seg_start[a], T.seg_len[a]
                assert any(g0 <= s and s + n <= g0 + ln for g0, ln, _ in runs)
    for r, p in enumerate(plans):
        runs = cqs.cqs_partial_runs(p, r, 0, N)
        held = sum(n for _, n, _ in runs)
        assert held <= p.info().acc_rows < held + cqs.CQS_ACC_BLOCK_ROWS * (len(runs) + 1)
        local = 0
        for g0, n, l0 in runs:   # packed in increasing global order
            assert l0 == local or l0 >= local
            local = l0 + n
        assert [pp.task(t).rank for pp in (p,) for t in range(info.n_tasks)] == owner


def test_contiguous_c4_fits_every_rank_and_shrinks_accumulators():
    """C4 at world 8: contiguous DFS runs keep each rank's held rows <= 0.7 N, so the resident
    replica (103 GB) + accumulator + output shard stays <= 170 GB on every rank (LPT: ~176 GB)."""
    N = 1 << 24
    for shard, lim in (("contiguous", 170e9), ("lpt", 180e9)):
        worst = max(cqs.cqs_plan(N=N, B=1, H=8, D=128, depth=3, world=8, rank=r,
                                 shard=shard).info().predicted_peak_bytes for r in range(8))
        assert worst <= lim
    accs = [cqs.cqs_plan(N=N, B=1, H=8, D=128, depth=3, world=8, rank=r,
                         shard="contiguous").info().acc_rows for r in range(8)]
    assert max(accs) <= 0.7 * N
    # streamed per rank: staging + accumulator + shard, far below the device
    ps = cqs.cqs_plan(N=N, B=1, H=8, D=128, depth=3, world=2, rank=0, shard="contiguous",
                      qkv_loc="host", out_loc="host")
    assert ps.info().predicted_peak_bytes <= 110e9 and ps.info().n_stage_buffers == 2


def test_contiguous_balance_c4():
    N = 1 << 24
    for world, tol in ((2, 1.005), (4, 1.01), (8, 1.03)):
        w = [cqs.cqs_plan(N=N, B=1, H=1, D=128, depth=3, world=world, rank=r,
                          shard="contiguous").info().my_work_pairs for r in range(world)]
        assert max(w) <= tol * N * N / world

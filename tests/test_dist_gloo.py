"""World-size-2 CPU (gloo) coverage of the multi-GPU path's host logic:
the C++ planner's LPT task assignment, the row shards, and the all-to-all exchange layout.
Each rank computes the partials of ITS tasks with the oracle (the GPU kernels need a device), the
exchange runs through paper_2604_20819_b200.dist over gloo, and the owner merges its shard with the
oracle's LSE merge; the union of shards must equal dense attention."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

I = (0, 1, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, H, D, depth, outdir, shard="lpt", qkv_loc="device"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from paper_2604_20819_b200 import dist as cdist
    from oracle import cqs_oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, k, v = (cqs_synth.numpy_tensor((1, H, N, D), 77, n) for n in ("q", "k", "v"))
    plan = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=depth, in_dtype="f32", world=world, rank=rank,
                        shard=shard, qkv_loc=qkv_loc, out_loc="host" if qkv_loc == "host" else None)
    info = plan.info()
    # this rank's rank-local accumulator: the rows cqs_partial_runs says it holds, in local order
    runs = cqs.cqs_partial_runs(plan, rank, 0, N)
    local_of = np.full(N, -1)
    for g0, n, l0 in runs:
        local_of[g0:g0 + n] = np.arange(l0, l0 + n)
    assert info.acc_rows >= (local_of.max() + 1) and info.acc_rows % cqs.CQS_ACC_BLOCK_ROWS == 0
    acc_o = np.zeros((info.acc_rows, H, D))
    acc_l = np.full((info.acc_rows, H), -np.inf)
    mine = 0
    for t in range(info.n_tasks):
        task = plan.task(t)
        if task.rank != rank:
            continue
        mine += 1
        e = O.build_subseq_entry(N, 7, I, tuple(task.quorum[i] for i in range(depth)))
        Oi, li = O.task_partial(q, k, v, e)
        rows_kept = np.isfinite(li[0, 0])          # query rows with a kept key
        idx = local_of[e.token_ids[rows_kept]]
        assert (idx >= 0).all(), "a task's query row is not in its rank's accumulator"
        mo, ml = O.lse_merge([(acc_o[idx], acc_l[idx]),
                              (Oi[0].transpose(1, 0, 2)[rows_kept], li[0].transpose(1, 0)[rows_kept])])
        acc_o[idx], acc_l[idx] = mo, ml
    assert mine == info.my_tasks
    ro, rl, part_off, part_row0 = cdist.exchange_partials(
        plan, torch.from_numpy(acc_o.reshape(-1, H * D)), torch.from_numpy(acc_l))
    row0, rows = cqs.cqs_shard_rows(N, world, rank)
    # owner side (the GPU's cqs_exchange_merge, here with the oracle merge): per global row of the
    # shard, the partials of every rank holding it
    parts = [[] for _ in range(rows)]
    for r in range(world):
        for g0, n, l0 in cqs.cqs_partial_runs(plan, r, row0, rows):
            for i in range(n):
                x = part_off[r] + (l0 + i - part_row0[r])
                parts[g0 + i - row0].append((ro[x].numpy().reshape(H, D), rl[x].numpy()))
    Om = np.zeros((rows, H, D))
    lm = np.zeros((rows, H))
    for i, ps in enumerate(parts):
        assert ps, "row %d held by no rank" % (row0 + i)
        Om[i], lm[i] = O.lse_merge(ps)
    np.save(os.path.join(outdir, "o%d.npy" % rank), Om)
    np.save(os.path.join(outdir, "l%d.npy" % rank), lm)
    np.save(os.path.join(outdir, "w%d.npy" % rank),
            np.array([info.my_work_pairs, row0, rows, info.acc_rows]))
    dist.destroy_process_group()


@pytest.mark.parametrize("shard,qkv_loc", [("lpt", "device"), ("contiguous", "device"),
                                           ("contiguous", "host")])
@pytest.mark.parametrize("N,depth", [(343, 3), (448, 1), (1030, 2), (2500, 3)])
def test_two_rank_exchange_reproduces_dense(N, depth, shard, qkv_loc, tmp_path):
    """Rank-local accumulators (held blocks only) + one all-to-all exchange over gloo: each owner's
    shard equals dense attention; resident and streamed plans, LPT and contiguous sharding."""
    import cqs_synth
    from oracle import cqs_oracle as O
    world, H, D = 2, 2, 32
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), shard,
                                      qkv_loc),
                       nprocs=world, start_method="fork")
    q, k, v = (cqs_synth.numpy_tensor((1, H, N, D), 77, n) for n in ("q", "k", "v"))
    Od, ld = O.dense_attention(q, k, v)
    Od = Od[0].transpose(1, 0, 2)
    ld = ld[0].transpose(1, 0)
    tot_work = 0
    for r in range(world):
        w, row0, rows, acc_rows = np.load(tmp_path / ("w%d.npy" % r))
        tot_work += w
        Om = np.load(tmp_path / ("o%d.npy" % r))
        lm = np.load(tmp_path / ("l%d.npy" % r))
        assert np.abs(Om - Od[row0:row0 + rows]).max() < 1e-12
        assert np.abs(lm - ld[row0:row0 + rows]).max() < 1e-12
    assert tot_work == N * N


@pytest.mark.parametrize("world", [3, 4])
@pytest.mark.parametrize("N,depth,shard,qkv_loc", [(1030, 2, "lpt", "device"),
                                                   (2500, 3, "contiguous", "device"),
                                                   (2401, 3, "contiguous", "host")])
def test_multi_rank_exchange_reproduces_dense(world, N, depth, shard, qkv_loc, tmp_path):
    """The same data plane at 3 and 4 ranks (ragged row shards at 3): every task on exactly one
    rank, every row held by some rank, each owner's merged shard equals dense attention."""
    import cqs_synth
    from oracle import cqs_oracle as O
    H, D = 2, 32
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), shard,
                                      qkv_loc),
                       nprocs=world, start_method="fork")
    q, k, v = (cqs_synth.numpy_tensor((1, H, N, D), 77, n) for n in ("q", "k", "v"))
    Od, ld = O.dense_attention(q, k, v)
    Od = Od[0].transpose(1, 0, 2)
    ld = ld[0].transpose(1, 0)
    tot_work, covered = 0, 0
    for r in range(world):
        w, row0, rows, acc_rows = np.load(tmp_path / ("w%d.npy" % r))
        assert row0 == covered
        covered += rows
        tot_work += w
        Om = np.load(tmp_path / ("o%d.npy" % r))
        lm = np.load(tmp_path / ("l%d.npy" % r))
        assert np.abs(Om - Od[row0:row0 + rows]).max() < 1e-12
        assert np.abs(lm - ld[row0:row0 + rows]).max() < 1e-12
    assert covered == N and tot_work == N * N


def _bwd_worker(rank, world, port, N, H, D, depth, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from paper_2604_20819_b200 import dist as cdist
    from oracle import cqs_oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, k, v, do = (cqs_synth.numpy_tensor((1, H, N, D), 78, n) for n in ("q", "k", "v", "do"))
    plan = cqs.cqs_plan(N=N, B=1, H=H, D=64, depth=depth, in_dtype="bf16", world=world, rank=rank)
    info = plan.info()   # (the planner's task sharding does not depend on D; D=16 keeps it small)
    entries, mine = [], set()
    for t in range(info.n_tasks):
        task = plan.task(t)
        entries.append(O.build_subseq_entry(N, 7, I, tuple(task.quorum[i] for i in range(depth))))
        if task.rank == rank:
            mine.add(t)
    grads = O.cqsa_backward_alg2(q, k, v, do, entries, only=mine)   # this rank's partials
    out = []
    for g in grads:   # token-major [N, H*D] like cqs_backward_partial_view
        acc = torch.from_numpy(np.ascontiguousarray(g[0].transpose(1, 0, 2).reshape(N, H * D)))
        recv, row0, rows = cdist.exchange_rows(acc, N, world, rank)
        out.append(sum(recv[r * rows:(r + 1) * rows].numpy() for r in range(world)))
    np.save(os.path.join(outdir, "g%d.npy" % rank), np.stack(out))
    np.save(os.path.join(outdir, "s%d.npy" % rank), np.array([row0, rows, len(mine)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("N,depth", [(343, 2), (500, 1)])
def test_two_rank_backward_exchange_reproduces_dense_grads(N, depth, tmp_path):
    """Task-sharded backward: each rank IndexAdds only its LPT tasks' gradients (Alg. 2 loop
    P:114-124 split across ranks), the owner sums the exchanged rows; the union equals the dense
    gradients."""
    import cqs_synth
    from oracle import cqs_oracle as O
    world, H, D = 2, 2, 16
    mp.start_processes(_bwd_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path)),
                       nprocs=world, start_method="fork")
    q, k, v, do = (cqs_synth.numpy_tensor((1, H, N, D), 78, n) for n in ("q", "k", "v", "do"))
    ref = [g[0].transpose(1, 0, 2).reshape(N, H * D) for g in O.dense_attention_grads(q, k, v, do)]
    ntasks = 0
    for r in range(world):
        row0, rows, nt = np.load(tmp_path / ("s%d.npy" % r))
        ntasks += nt
        got = np.load(tmp_path / ("g%d.npy" % r))
        for g, rf in zip(got, ref):
            assert np.abs(g - rf[row0:row0 + rows]).max() < 1e-10
    assert ntasks == 7 ** depth

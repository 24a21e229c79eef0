"""Two ranks sharing cuda:0 (the round's GPU budget is one device): each rank runs
cqs_attention_forward on ITS LPT-assigned tasks (world=2 plan), the partial accumulators are
exchanged with paper_2604_20819_b200.dist over gloo (CPU copies; NCCL refuses two ranks on one
device), and each owner merges its row shard with the cqs_merge kernel.  The union of shards must
match the fp64 oracle — this exercises the multi-GPU product path except the NCCL transport."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, H, D, depth, outdir, mode="gloo", schedule="uniform",
            shard="lpt", qkv_loc="device", dtype="bf16", n_parallel=0):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from paper_2604_20819_b200 import dist as cdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 4242, dtype=tdt, device="cuda")
    streamed = qkv_loc == "host"
    if streamed:   # each rank stages only its tasks' segments from pinned host memory
        q, k, v = (t.cpu().pin_memory() for t in (q, k, v))
    plan = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=depth, in_dtype=dtype, world=world, rank=rank,
                        schedule=schedule, shard=shard, qkv_loc=qkv_loc,
                        out_loc="host" if streamed else "device", n_parallel=n_parallel)
    info = plan.info()
    dev_bytes, host_bytes = cqs.cqs_forward_workspace_size(plan)
    assert host_bytes == 0
    ws = torch.empty(dev_bytes, dtype=torch.uint8, device="cuda")
    row0, rows = cqs.cqs_shard_rows(N, world, rank)
    assert info.shard_rows == rows
    out = torch.zeros(1, H, rows, D, dtype=tdt, device="cuda")   # owned shard only
    lse = torch.zeros(1, H, rows, dtype=torch.float32, device="cuda")
    cqs.cqs_attention_forward(plan, q, k, v, None, None, 0.0, 0, ws, None)
    torch.cuda.synchronize()
    if mode == "p2p":   # exchange + merge over peer (IPC-mapped) memory
        px = cdist.PeerExchange(plan, ws)
        px.merge(out, lse)
        px.close()
    else:               # all-to-all (gloo: CPU copies) + cqs_exchange_merge on the GPU
        acc_o, acc_l = cdist.partial_accumulator(plan, ws)
        ro, rl, off, pr0 = cdist.exchange_partials(plan, acc_o.cpu(), acc_l.cpu())
        cdist.merge_received(plan, ro.cuda(), rl.cuda(), off, pr0, out, lse)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, "o%d.npy" % rank), out[0].float().cpu().numpy())
    np.save(os.path.join(outdir, "l%d.npy" % rank), lse[0].cpu().numpy())
    np.save(os.path.join(outdir, "s%d.npy" % rank), np.array([row0, rows, info.acc_rows]))
    dist.destroy_process_group()


def _check_shards(tmp_path, world, N, H, D, seed=4242, dtype=torch.bfloat16, tol=2e-2,
                  ltol=1e-3):
    import cqs_synth
    from oracle import cqs_oracle as O
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, seed, dtype=dtype)
    if N <= 6000:
        Od, ld = O.dense_attention(*(t.double().numpy() for t in (q, k, v)))
    rng = np.random.default_rng(N)
    for r in range(world):
        row0, rows, _ = np.load(tmp_path / ("s%d.npy" % r))
        o = np.load(tmp_path / ("o%d.npy" % r))
        l_ = np.load(tmp_path / ("l%d.npy" % r))
        if N <= 6000:
            ref = Od[0, :, row0:row0 + rows]
            err = np.abs(o - ref).max()
            # bf16: absolute (R16); fp32: normwise relative (R15)
            assert err <= (tol if dtype == torch.bfloat16 else tol * np.abs(ref).max()), err
            assert np.abs(l_ - ld[0, :, row0:row0 + rows]).max() <= ltol
            continue
        # sampled rows: both shard edges plus random rows, every head
        sel = np.unique(np.concatenate([[0, rows - 1], rng.choice(rows, 150, replace=False)]))
        for h in range(H):
            Oref, lref = O.dense_attention_rows(*(t[0, h].double().numpy() for t in (q, k, v)),
                                                row0 + sel)
            assert np.abs(o[h, sel] - Oref).max() <= 2e-2
            assert np.abs(l_[h, sel] - lref).max() <= 1e-3


@pytest.mark.parametrize("mode,schedule,shard", [("gloo", "uniform", "lpt"),
                                                 ("p2p", "uniform", "lpt"),
                                                 ("p2p", "hybrid", "lpt"),
                                                 ("p2p", "uniform", "contiguous"),
                                                 ("gloo", "uniform", "contiguous")])
@pytest.mark.parametrize("N,depth", [(3000, 2), (2401, 3), (5000, 1)])
def test_two_ranks_one_gpu(N, depth, mode, schedule, shard, tmp_path):
    world, H, D = 2, 2, 128
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), mode,
                                      schedule, shard),
                       nprocs=world, start_method="spawn")
    _check_shards(tmp_path, world, N, H, D)


@pytest.mark.parametrize("mode", ["p2p", "gloo"])
@pytest.mark.parametrize("N,depth,D", [(20000, 3, 128), (12000, 4, 64)])
def test_two_ranks_streamed_c4_shape(N, depth, D, mode, tmp_path):
    """C4's multi-rank layout at small N: Q/K/V in pinned host memory, every rank stages only its
    (contiguous) tasks' segments, keeps a rank-local accumulator, and one exchange finalizes the
    owned shards."""
    world, H = 2, 2
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), mode,
                                      "uniform", "contiguous", "host"),
                       nprocs=world, start_method="spawn")
    _check_shards(tmp_path, world, N, H, D)


def _bwd_worker(rank, world, port, N, H, D, depth, outdir, mode, schedule="uniform"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from paper_2604_20819_b200 import dist as cdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 4243, dtype=torch.bfloat16, device="cuda")
    do = cqs_synth.torch_tensor((1, H, N, D), 4243, "do", torch.bfloat16, "cuda")
    out, lse = cqs.attention(q, k, v, depth=depth)     # O, lse on every rank (as after all-gather)
    plan = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=depth, in_dtype="bf16", out_dtype="f32",
                        world=world, rank=rank, schedule=schedule)
    bws = torch.empty(cqs.cqs_backward_workspace_size(plan), dtype=torch.uint8, device="cuda")
    cqs.cqs_attention_backward(plan, q, k, v, out, do, lse, None, None, None, 0.0, bws)
    torch.cuda.synchronize()
    grads = [torch.zeros(1, H, N, D, dtype=torch.float32, device="cuda") for _ in range(3)]
    if mode == "p2p":
        pr = cdist.PeerGradReduce(plan, bws, N, 1, H, D, world, rank)
        row0, rows = pr.row0, pr.rows
        pr.reduce(*grads)
        pr.close()
    else:
        base = bws.data_ptr()
        for addr, g in zip(cqs.cqs_backward_partial_view(plan, bws), grads):
            acc = bws[addr - base: addr - base + N * H * D * 4].view(torch.float32).view(N, H * D)
            recv, row0, rows = cdist.exchange_rows(acc.cpu(), N, world, rank)
            cdist.reduce_grads_gpu(recv.cuda(), world, rows, 1, H, D, g, row0)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, "g%d.npy" % rank),
            np.stack([g[0, :, row0:row0 + rows].cpu().numpy() for g in grads]))
    np.save(os.path.join(outdir, "s%d.npy" % rank), np.array([row0, rows]))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,schedule", [("gloo", "uniform"), ("p2p", "uniform"),
                                           ("p2p", "hybrid")])
@pytest.mark.parametrize("N,depth", [(3000, 2), (1030, 1)])
def test_two_ranks_backward_one_gpu(N, depth, mode, schedule, tmp_path):
    """Task-sharded backward (each rank its LPT tasks) + one exchange: the owners' row shards of
    dQ/dK/dV match the oracle's dense gradients within R19."""
    import cqs_synth
    from oracle import cqs_oracle as O
    world, H, D = 2, 2, 128
    mp.start_processes(_bwd_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), mode,
                                          schedule),
                       nprocs=world, start_method="spawn")
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 4243, dtype=torch.bfloat16)
    do = cqs_synth.torch_tensor((1, H, N, D), 4243, "do", torch.bfloat16)
    ref = O.dense_attention_grads(*(t.double().numpy() for t in (q, k, v, do)))
    for r in range(world):
        row0, rows = np.load(tmp_path / ("s%d.npy" % r))
        got = np.load(tmp_path / ("g%d.npy" % r))
        for g, rf in zip(got, ref):
            rf = rf[0, :, row0:row0 + rows]
            assert np.linalg.norm(g - rf) / np.linalg.norm(rf) <= 1e-2


@pytest.mark.parametrize("mode,shard,qkv_loc", [("p2p", "contiguous", "device"),
                                                ("gloo", "lpt", "host")])
def test_two_ranks_f32(mode, shard, qkv_loc, tmp_path):
    """The fp32 path (BASELINE config 0's dtype) through the multi-rank data plane: rank-local
    accumulators, streamed or resident, one exchange; R15 tolerance (1e-5 relative)."""
    world, N, H, D, depth = 2, 1500, 2, 64, 2
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), mode,
                                      "uniform", shard, qkv_loc, "f32"),
                       nprocs=world, start_method="spawn")
    _check_shards(tmp_path, world, N, H, D, dtype=torch.float32, tol=1e-5, ltol=1e-5)


def test_two_ranks_parallel_slots(tmp_path):
    """world 2 with 3 tasks in flight per rank: the slots are folded into the rank-local
    accumulator before the exchange reads it."""
    world, N, H, D, depth = 2, 3000, 2, 128, 3
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), "p2p",
                                      "uniform", "contiguous", "device", "bf16", 3),
                       nprocs=world, start_method="spawn")
    _check_shards(tmp_path, world, N, H, D)

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


def _worker(rank, world, port, N, H, D, depth, outdir, mode="gloo", schedule="uniform"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import cqs_synth
    import paper_2604_20819_b200 as cqs
    from paper_2604_20819_b200 import dist as cdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 4242, dtype=torch.bfloat16, device="cuda")
    plan = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=depth, in_dtype="bf16", world=world, rank=rank,
                        schedule=schedule)
    dev_bytes, _ = cqs.cqs_forward_workspace_size(plan)
    ws = torch.empty(dev_bytes, dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, H, N, D, dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(1, H, N, dtype=torch.float32, device="cuda")
    cqs.cqs_attention_forward(plan, q, k, v, out, None, 0.0, 0, ws, None)
    ao, al = cqs.cqs_partial_view(plan, ws)
    base = ws.data_ptr()
    acc_o = ws[ao - base: ao - base + N * H * D * 4].view(torch.float32).view(N, H * D)
    acc_l = ws[al - base: al - base + N * H * 4].view(torch.float32).view(N, H)
    torch.cuda.synchronize()
    if mode == "p2p":   # exchange + merge in one kernel over peer (IPC-mapped) memory
        px = cdist.PeerExchange(plan, ws, N, 1, H, D, world, rank)
        row0, rows = px.row0, px.rows
        px.merge(out, lse)
        px.close()
    else:
        ro, rl, row0, rows = cdist.exchange_partials(acc_o.cpu(), acc_l.cpu(), N, world, rank)
        cdist.merge_shard_gpu(ro.cuda(), rl.cuda(), world, rows, 1, H, D, out, lse, row0, N)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, "o%d.npy" % rank), out[0, :, row0:row0 + rows].float().cpu().numpy())
    np.save(os.path.join(outdir, "l%d.npy" % rank), lse[0, :, row0:row0 + rows].cpu().numpy())
    np.save(os.path.join(outdir, "s%d.npy" % rank), np.array([row0, rows]))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,schedule", [("gloo", "uniform"), ("p2p", "uniform"),
                                           ("p2p", "hybrid")])
@pytest.mark.parametrize("N,depth", [(3000, 2), (2401, 3), (5000, 1)])
def test_two_ranks_one_gpu(N, depth, mode, schedule, tmp_path):
    import cqs_synth
    from oracle import cqs_oracle as O
    world, H, D = 2, 2, 128
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, depth, str(tmp_path), mode,
                                      schedule),
                       nprocs=world, start_method="spawn")
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 4242, dtype=torch.bfloat16)
    Od, ld = O.dense_attention(*(t.double().numpy() for t in (q, k, v)))
    for r in range(world):
        row0, rows = np.load(tmp_path / ("s%d.npy" % r))
        o = np.load(tmp_path / ("o%d.npy" % r))
        l_ = np.load(tmp_path / ("l%d.npy" % r))
        assert np.abs(o - Od[0, :, row0:row0 + rows]).max() <= 2e-2
        assert np.abs(l_ - ld[0, :, row0:row0 + rows]).max() <= 1e-3


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

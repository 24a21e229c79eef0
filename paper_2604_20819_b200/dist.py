"""Multi-GPU exchange for task-sharded CQS attention.

Every rank runs `cqs_attention_forward` on the tasks its plan assigns to it (LPT or contiguous DFS
runs on exact work, no communication during compute).  Each rank's fp32 partial accumulator holds
only the rows its tasks touch (`cqs_partial_view`, `cqs_partial_runs`) and is exchanged ONCE: the
owner of each contiguous row shard (`cqs_shard_rows`) LSE-merges the partials of the ranks holding
each of its rows (`cqs_exchange_merge` on the GPU), reading them over peer memory
(`PeerExchange`) or from an all-to-all (`exchange_partials` + `merge_received`).
torch.distributed is the transport (NCCL on GPUs, gloo in CPU tests): plumbing only — no
arithmetic happens here.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import cqs_backward_partial_view, cqs_exchange_merge, cqs_ipc_close, cqs_ipc_handle, \
    cqs_ipc_open, cqs_partial_runs, cqs_partial_view, cqs_reduce_sum, cqs_shard_rows


def shard_spans(N: int, world: int):
    """[(row0, rows)] per rank (the owner shards of the final merge)."""
    return [cqs_shard_rows(N, world, r) for r in range(world)]


def partial_span(plan, src_rank: int, row0: int, rows: int):
    """(first local row, row count) of rank src_rank's accumulator rows inside the global rows
    [row0, row0+rows) — one contiguous local range (held blocks are packed in global order)."""
    runs = cqs_partial_runs(plan, src_rank, row0, rows)
    if not runs:
        return 0, 0
    return runs[0][2], sum(n for _, n, _ in runs)


def partial_accumulator(plan, ws):
    """This rank's fp32 accumulator inside the forward workspace as tensors
    ([acc_rows, B*H*D], [acc_rows, B*H])."""
    d = plan.desc
    BH, D, rows = d.B * d.H, d.D, plan.info().acc_rows
    ao, al = cqs_partial_view(plan, ws)
    base = ws.data_ptr()
    acc_o = ws[ao - base: ao - base + rows * BH * D * 4].view(torch.float32).view(rows, BH * D)
    acc_l = ws[al - base: al - base + rows * BH * 4].view(torch.float32).view(rows, BH)
    return acc_o, acc_l


def exchange_partials(plan, acc_o: torch.Tensor, acc_l: torch.Tensor, group=None):
    """The all-to-all transport of the exchange step: every rank sends each owner the rows of its
    accumulator that fall into the owner's shard (a contiguous local range each, in shard order).
    acc_o / acc_l: this rank's accumulator ([acc_rows, B*H*D] / [acc_rows, B*H], any device the
    process group's backend handles).  Returns (recv_o, recv_l, part_off, part_row0): the received
    rows, rank-major; part_off[r] = first received row from rank r; part_row0[r] = the local
    accumulator row of rank r that chunk starts at (cqs_exchange_merge's part_row0)."""
    d = plan.desc
    world, rank, N = d.world, d.rank, d.N
    spans = shard_spans(N, world)
    send = [partial_span(plan, rank, r0, n) for r0, n in spans]
    first = next((a for a, c in send if c), 0)
    assert all(a == first + sum(c for _, c in send[:i]) for i, (a, c) in enumerate(send) if c)
    tot = sum(c for _, c in send)
    row0, rows = spans[rank]
    recv = [partial_span(plan, r, row0, rows) for r in range(world)]
    in_splits = [c for _, c in send]
    out_splits = [c for _, c in recv]
    recv_o = acc_o.new_empty((sum(out_splits), acc_o.shape[1]))
    recv_l = acc_l.new_empty((sum(out_splits), acc_l.shape[1]))
    dist.all_to_all_single(recv_o, acc_o[first:first + tot].contiguous(), out_splits, in_splits,
                           group=group)
    dist.all_to_all_single(recv_l, acc_l[first:first + tot].contiguous(), out_splits, in_splits,
                           group=group)
    part_off, off = [], 0
    for c in out_splits:
        part_off.append(off)
        off += c
    return recv_o, recv_l, part_off, [a for a, _ in recv]


def merge_received(plan, recv_o, recv_l, part_off, part_row0, out, lse=None, stream=None):
    """Owner-side merge of the all-to-all buffers into its shard (cqs_exchange_merge kernel(s)).
    out: device [B,H,shard_rows,D]; lse: device fp32 [B,H,shard_rows] or None."""
    wo = recv_o.shape[1] * 4
    wl = recv_l.shape[1] * 4
    po = [recv_o.data_ptr() + o * wo for o in part_off]
    pl = [recv_l.data_ptr() + o * wl for o in part_off]
    cqs_exchange_merge(plan, po, pl, part_row0, out, lse, stream)


class PeerExchange:
    """Exchange + merge over peer memory (NVLink / NVSwitch): every rank maps all ranks'
    rank-local accumulators (CUDA IPC, handles swapped once through torch.distributed) and the
    owner's cqs_exchange_merge reads the holders' rows of its shard directly over the links — no
    staging all-to-all, no second pass.  The workspace must stay allocated (and at the same
    address) for the object's lifetime; mappings are reused across steps."""

    def __init__(self, plan, ws, group=None):
        d = plan.desc
        self.plan, self.world, self.rank, self.group = plan, d.world, d.rank, group
        ao, al = cqs_partial_view(plan, ws)
        mine = (cqs_ipc_handle(ao), cqs_ipc_handle(al))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self.opened = []
        self.po, self.pl = [], []
        self.row0, self.rows = cqs_shard_rows(d.N, self.world, self.rank)
        for r in range(self.world):
            if r == self.rank:
                bo, bl = ao, al
            else:
                (ho, oo), (hl, ol) = allh[r]
                base_o = cqs_ipc_open(ho)
                self.opened.append(base_o)
                if hl == ho:                      # same allocation (one workspace tensor)
                    base_l = base_o
                else:
                    base_l = cqs_ipc_open(hl)
                    self.opened.append(base_l)
                bo, bl = base_o + oo, base_l + ol
            self.po.append(bo)
            self.pl.append(bl)

    def merge(self, out, lse=None, stream=None):
        """Call after every rank's forward has been issued on its stream: barrier (all partials
        complete), the owner's merge over peer memory, barrier (peers done reading).
        out: device [B,H,shard_rows,D]; lse: device fp32 [B,H,shard_rows] or None."""
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        dist.barrier(group=self.group)
        cqs_exchange_merge(self.plan, self.po, self.pl, [0] * self.world, out, lse, stream)
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        dist.barrier(group=self.group)

    def close(self):
        for b in self.opened:
            cqs_ipc_close(b)
        self.opened = []


# ------------------------------------------------------------------------------------------------
# Backward (Algorithm 2, NEXT-1) across ranks: every rank accumulates the gradients of ITS tasks
# into full-size fp32 [N][B*H][D] partials (cqs_backward_partial_view); the owner of each row shard
# sums the ranks' rows (Alg. 2's IndexAdd, done across GPUs) with cqs_reduce_sum.
# ------------------------------------------------------------------------------------------------

def exchange_rows(acc: torch.Tensor, N: int, world: int, rank: int, group=None):
    """acc: [N, W] partial of this rank.  Returns ([world*rows, W] rank-major rows of this rank's
    shard from every rank, row0, rows) — the all-to-all transport (NCCL on GPUs, gloo on CPU)."""
    spans = shard_spans(N, world)
    row0, rows = spans[rank]
    recv = acc.new_empty((world * rows, acc.shape[1]))
    dist.all_to_all_single(recv, acc.contiguous(), [rows] * world, [n for _, n in spans],
                           group=group)
    return recv, row0, rows


def reduce_grads_gpu(recv, world, rows, B, H, D, out, row0, stream=None):
    """Sum the received rank-major partial rows into rows [row0, row0+rows) of `out`."""
    cqs_reduce_sum(rows, B, H, D, [recv[r * rows:(r + 1) * rows] for r in range(world)], out,
                   out_row0=row0, stream=stream)


class PeerGradReduce:
    """Backward exchange + sum in one kernel per gradient over peer memory: every rank maps all
    ranks' dQ/dK/dV partial accumulators (CUDA IPC, handles swapped once) and sums the peers' rows
    of its shard directly over NVLink / NVSwitch into its dQ/dK/dV.  The backward workspace must
    stay allocated (same address) for the object's lifetime."""

    def __init__(self, plan, bws, N, B, H, D, world, rank, group=None):
        self.N, self.B, self.H, self.D, self.world, self.rank = N, B, H, D, world, rank
        self.group = group
        views = cqs_backward_partial_view(plan, bws)
        mine = [cqs_ipc_handle(a) for a in views]
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.row0, self.rows = cqs_shard_rows(N, world, rank)
        self.opened = []
        self.parts = [[], [], []]          # per gradient: one address per rank
        BH = B * H
        for r in range(world):
            bases = {}
            for g in range(3):
                if r == rank:
                    addr = views[g]
                else:
                    h, off = allh[r][g]
                    if h not in bases:
                        bases[h] = cqs_ipc_open(h)
                        self.opened.append(bases[h])
                    addr = bases[h] + off
                self.parts[g].append(addr + self.row0 * BH * D * 4)

    def reduce(self, dq, dk, dv, stream=None):
        """After every rank's backward was issued: barrier, three sum kernels reading the peers'
        rows over NVLink, barrier (peers done reading before the workspace is reused)."""
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        dist.barrier(group=self.group)
        for g, out in enumerate((dq, dk, dv)):
            cqs_reduce_sum(self.rows, self.B, self.H, self.D, self.parts[g], out,
                           out_row0=self.row0, stream=stream)
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        dist.barrier(group=self.group)

    def close(self):
        for b in self.opened:
            cqs_ipc_close(b)
        self.opened = []

"""Multi-GPU exchange for task-sharded CQS attention.

Every rank runs `cqs_attention_forward` on the tasks its plan assigns to it (LPT on exact work, no
communication during compute).  Each rank's fp32 partial accumulator ([N][B*H][D] + [N][B*H], see
`cqs_partial_view`) is then exchanged ONCE: all-to-all of partial rows to the owner of each
contiguous row shard (`cqs_shard_rows`), after which the owner LSE-merges the R partials of its rows
(`cqs_merge` on the GPU).  torch.distributed is the transport (NCCL on GPUs, gloo in CPU tests):
plumbing only — no arithmetic happens here.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import cqs_backward_partial_view, cqs_ipc_close, cqs_ipc_handle, cqs_ipc_open, cqs_merge, \
    cqs_partial_view, cqs_reduce_sum, cqs_shard_rows


def shard_spans(N: int, world: int):
    """[(row0, rows)] per rank (the owner shards of the final merge)."""
    return [cqs_shard_rows(N, world, r) for r in range(world)]


def exchange_partials(acc_o: torch.Tensor, acc_l: torch.Tensor, N: int, world: int, rank: int,
                      group=None):
    """acc_o: [N, B*H*D] fp32 partial of this rank; acc_l: [N, B*H].  Returns (recv_o, recv_l,
    row0, rows): the partials of this rank's shard from every rank, rank-major
    ([world*rows, B*H*D] and [world*rows, B*H])."""
    spans = shard_spans(N, world)
    row0, rows = spans[rank]
    in_splits = [n for _, n in spans]
    out_splits = [rows] * world
    recv_o = acc_o.new_empty((world * rows, acc_o.shape[1]))
    recv_l = acc_l.new_empty((world * rows, acc_l.shape[1]))
    dist.all_to_all_single(recv_o, acc_o.contiguous(), out_splits, in_splits, group=group)
    dist.all_to_all_single(recv_l, acc_l.contiguous(), out_splits, in_splits, group=group)
    return recv_o, recv_l, row0, rows


def split_parts(recv_o: torch.Tensor, recv_l: torch.Tensor, world: int, rows: int):
    """Per-rank views of the received partials, in rank order (fixed merge order)."""
    po = [recv_o[r * rows:(r + 1) * rows] for r in range(world)]
    pl = [recv_l[r * rows:(r + 1) * rows] for r in range(world)]
    return po, pl


def merge_shard_gpu(recv_o, recv_l, world, rows, B, H, D, out, lse, row0, N, stream=None):
    """R-way LSE merge of the received partials into rows [row0, row0+rows) of out / lse
    (cqs_merge kernel on the GPU)."""
    po, pl = split_parts(recv_o, recv_l, world, rows)
    cqs_merge(rows, B, H, D, po, pl, out=out, out_row0=row0, n_total=N, lse_out=lse,
              stream=stream)


class PeerExchange:
    """Exchange + merge in ONE kernel over peer memory (NVLink / NVSwitch): every rank maps all
    ranks' partial accumulators (CUDA IPC, handles swapped once through torch.distributed) and
    launches cqs_merge with the peers' shard rows as its parts, reading them directly over the
    links — no staging all-to-all, no second pass.  The workspace must stay allocated (and at the
    same address) for the object's lifetime; mappings are reused across steps."""

    def __init__(self, plan, ws, N, B, H, D, world, rank, group=None):
        self.N, self.B, self.H, self.D, self.world, self.rank = N, B, H, D, world, rank
        self.group = group
        ao, al = cqs_partial_view(plan, ws)
        mine = (cqs_ipc_handle(ao), cqs_ipc_handle(al))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.opened = []
        self.po, self.pl = [], []
        self.row0, self.rows = cqs_shard_rows(N, world, rank)
        BH = B * H
        for r in range(world):
            if r == rank:
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
            self.po.append(bo + self.row0 * BH * D * 4)
            self.pl.append(bl + self.row0 * BH * 4)

    def merge(self, out, lse, stream=None):
        """Call after every rank's forward has been issued on its stream: barrier (all partials
        complete), one merge kernel over peer memory, barrier (peers done reading)."""
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        dist.barrier(group=self.group)
        cqs_merge(self.rows, self.B, self.H, self.D, self.po, self.pl, out=out, out_row0=self.row0,
                  n_total=self.N, lse_out=lse, stream=stream)
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

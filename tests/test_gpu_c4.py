"""BASELINE config 3 (C4) at full size on one GPU: N = 2^24 tokens, H = 8, D = 128, bf16, depth 3
(343 tasks, 7 empty), plan sharded over world = 8 with contiguous task runs.  This
process runs rank 0's share into its rank-local accumulator (held blocks only, cqs_partial_runs) —
the memory layout that makes C4 fit one B200 per rank (resident replica 103 GB + accumulator
<= 0.7 N rows + output shard: cqs_plan predicts <= 170 GB for every rank) — and the accumulator is
checked on sampled rows of two heads against the oracle's partial over exactly rank 0's tasks
(literal Algorithm 3 entries; LSE merge)."""
import numpy as np
import pytest
import torch

import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
I = (0, 1, 3)


def test_c4_rank0_partial_sampled_rows():
    N, H, D, depth, world = 1 << 24, 8, 128, 3, 8
    for r in range(world):
        pr = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=depth, in_dtype="bf16", world=world, rank=r,
                          shard="contiguous")
        assert pr.info().predicted_peak_bytes <= 170e9
    q, k, v = cqs_synth.torch_qkv(1, H, N, D, 20260420, dtype=torch.bfloat16, device="cuda")
    plan = cqs.cqs_plan(N=N, B=1, H=H, D=D, depth=depth, in_dtype="bf16", world=world, rank=0,
                        shard="contiguous")
    info = plan.info()
    assert info.n_tasks == 343 and info.n_empty == 7 and info.acc_rows < 0.75 * N
    dev_bytes, _ = cqs.cqs_forward_workspace_size(plan)
    ws = torch.empty(dev_bytes, dtype=torch.uint8, device="cuda")
    cqs.cqs_attention_forward(plan, q, k, v, None, None, 0.0, 0, ws, None)
    torch.cuda.synchronize()
    ao, al = cqs.cqs_partial_view(plan, ws)
    base = ws.data_ptr()
    A = info.acc_rows
    acc_o = ws[ao - base: ao - base + A * H * D * 4].view(torch.float32).view(A, H, D)
    acc_l = ws[al - base: al - base + A * H * 4].view(torch.float32).view(A, H)
    local = {}
    for g0, n, l0 in cqs.cqs_partial_runs(plan, 0, 0, N):
        local[(g0, n)] = l0

    def local_row(g):
        for (g0, n), l0 in local.items():
            if g0 <= g < g0 + n:
                return l0 + g - g0
        return None

    rng = np.random.default_rng(3)
    held = [g for g in rng.choice(N, 400, replace=False) if local_row(int(g)) is not None]
    rows = np.sort(np.array(held[:10]))
    entries = []
    for t in range(info.n_tasks):
        task = plan.task(t)
        if task.rank == 0:
            entries.append(O.build_subseq_entry(N, 7, I, tuple(task.quorum[i] for i in range(depth))))
    alpha = 1 / np.sqrt(D)
    lrows = torch.tensor([local_row(int(n)) for n in rows]).cuda()
    for h in (0, H - 1):
        qn = q[0, h].float().cpu().numpy()
        kn = k[0, h].float().cpu().numpy()
        vn = v[0, h].float().cpu().numpy()
        parts = {int(r): [] for r in rows}
        for e in entries:
            for n in rows:
                hit = np.nonzero(e.token_ids == n)[0]
                if len(hit) == 0:
                    continue
                p = hit[0]
                keep = np.ones(len(e.token_ids), dtype=bool)
                for g in e.group_runs:                       # LocalMaskFromGroupRuns, row p
                    if any(s <= p < en for s, en in g):
                        for s, en in g:
                            keep[s:en] = False
                keys = e.token_ids[keep]
                if len(keys) == 0:
                    continue
                lg = alpha * (kn[keys].astype(np.float64) @ qn[n].astype(np.float64))
                mx = lg.max()
                w = np.exp(lg - mx)
                parts[int(n)].append(((w @ vn[keys].astype(np.float64)) / w.sum(),
                                      mx + np.log(w.sum())))
        got_o = acc_o[lrows, h].double().cpu().numpy()
        got_l = acc_l[lrows, h].double().cpu().numpy()
        for i, n in enumerate(rows):
            if not parts[int(n)]:
                assert np.isneginf(got_l[i])
                continue
            Om, lm = O.lse_merge([(o[None], np.array([l_])) for o, l_ in parts[int(n)]])
            assert np.abs(got_o[i] - Om[0]).max() <= 2e-2
            assert abs(got_l[i] - lm[0]) <= 1e-3
        del qn, kn, vn

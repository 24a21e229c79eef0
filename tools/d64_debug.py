"""Debug helper: D=64 kernel vs a torch fp32 reference at depth 0 for several KV lengths, with and
without growing key norms (rescale path).  Prints max |dO| and max |dlse| per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cqs_synth
import paper_2604_20819_b200 as cqs

D = int(os.environ.get("D", "64"))
for N in [256, 512, 640, 1280, 1408, 2560, 3000]:
    for ramp in (False, True):
        q, k, v = cqs_synth.torch_qkv(1, 2, N, D, 123 + D, dtype=torch.bfloat16, device="cuda")
        if ramp:
            r = torch.linspace(0.5, 4.0, N, device="cuda").view(1, 1, N, 1)
            k = (k.float() * r).to(torch.bfloat16)
        out, lse = cqs.attention(q, k, v, depth=0)
        s = (q.float() @ k.float().transpose(-1, -2)) / D ** 0.5
        ref = torch.softmax(s, -1) @ v.float()
        lref = torch.logsumexp(s, -1)
        e = (out.float() - ref).abs()
        bad = (e.amax(-1) > 2e-2).nonzero()
        print(N, ramp, "maxerr %.3e lse %.3e" % (e.max().item(), (lse - lref).abs().max().item()),
              "bad rows", bad.shape[0], bad[:6, -1].tolist())

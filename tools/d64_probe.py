"""Debug: per-row error of the D=64 kernel on the growing-logits workload (depth 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cqs_synth
import paper_2604_20819_b200 as cqs
from oracle import cqs_oracle as O
N, D = int(sys.argv[1]), 64
q, k, v = cqs_synth.torch_qkv(1, 1, N, D, 187, dtype=torch.bfloat16, device="cuda")
ramp = torch.linspace(0.5, 4.0, N, device="cuda").view(1, 1, N, 1)
k = (k.float() * ramp).to(torch.bfloat16)
out, lse = cqs.attention(q, k, v, depth=0)
torch.cuda.synchronize()
Od, ld = O.dense_attention(*(t.double().cpu().numpy() for t in (q, k, v)))
err = np.abs(out.double().cpu().numpy() - Od).max(axis=-1)[0, 0]
lerr = np.abs(lse.double().cpu().numpy() - ld)[0, 0]
bad = np.nonzero(err > 2e-2)[0]
print("bad rows", len(bad), bad[:20], "max err", err.max(), "lse err max", lerr.max(), "at", lerr.argmax())
print("bad rows mod 384:", np.unique(bad % 384)[:40])

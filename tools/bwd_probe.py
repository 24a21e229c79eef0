"""Debug helper for the backward: python tools/bwd_probe.py N D depth
Prints the prep buffer and the three fp32 accumulators against a plain torch fp32 reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cqs_synth
import paper_2604_20819_b200 as cqs

N, D, depth = (int(x) for x in sys.argv[1:4])
B, H = 1, 2
q, k, v = cqs_synth.torch_qkv(B, H, N, D, 1, dtype=torch.bfloat16, device="cuda")
do = cqs_synth.torch_tensor((B, H, N, D), 1, "do", torch.bfloat16, "cuda")
out, lse = cqs.attention(q, k, v, depth=depth)
p = cqs.cqs_plan(N=N, B=B, H=H, D=D, depth=depth, in_dtype="bf16", out_dtype="f32")
wsb = cqs.cqs_backward_workspace_size(p)
ws = torch.zeros(wsb // 4 + 64, dtype=torch.float32, device="cuda")
dq, dk, dv = (torch.empty((B, H, N, D), dtype=torch.float32, device="cuda") for _ in range(3))
cqs.cqs_attention_backward(p, q, k, v, out, do, lse, dq, dk, dv, 0.0, ws)
torch.cuda.synchronize()
pitch = (N + 3) // 4 * 4
ldb = ws[:B * H * 2 * pitch].view(B * H, 2, pitch)[:, :, :N]
a = 1 / D ** 0.5
qf, kf, vf, dof = (t.float() for t in (q, k, v, do))
S = a * qf @ kf.transpose(-1, -2)
P = torch.softmax(S, -1)
Of = P @ vf
delta = (dof * out.float()).sum(-1).reshape(B * H, N)
print("lse max err", float((ldb[:, 0] + lse.reshape(B * H, N) * 1.4426950408889634).abs().max()))
print("delta max err", float((ldb[:, 1] - delta).abs().max()), float(delta.abs().max()))
dV = P.transpose(-1, -2) @ dof
dP = dof @ vf.transpose(-1, -2)
dS = P * (dP - (dof * Of).sum(-1, keepdim=True))
dQ = a * dS @ kf
dK = a * dS.transpose(-1, -2) @ qf
for nm, g, r in (("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
    nan = int(torch.isnan(g).sum())
    bad = torch.isnan(g).any(-1)[0]
    rows = bad.nonzero()[:, 1][:10].tolist() if nan else []
    err = (g - r).nan_to_num(1e9)
    print(nm, "nan", nan, "rows", rows, "rel", float(err.norm() / r.norm()),
          "rowrel max", float((err.norm(dim=-1) / r.norm(dim=-1)).max()))

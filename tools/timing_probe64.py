"""Cycle accounting of the double-buffered-S D=64 kernel (debug build with -DCQS_DBG_TIMING, loaded
via CQS_LIB).  Counters: 0 softmax wait-for-S, 1 softmax S->P (incl. pair barrier), 2 softmax
steps (per warp), 3 pair-barrier wait, 4 MMA wait-for-P, 5 MMA total, 6 MMA kv-iterations,
7 MMA wait for K/V tiles."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cqs_synth
import paper_2604_20819_b200 as cqs

L = cqs.lib()
q, k, v = cqs_synth.torch_qkv(1, 32, 131072, 64, 20260418, dtype=torch.bfloat16, device="cuda")
cqs.attention(q, k, v, depth=1)
torch.cuda.synchronize()
L.cqs_dbg64_reset()
cqs.attention(q, k, v, depth=1)
torch.cuda.synchronize()
c = (ctypes.c_ulonglong * 16)()
L.cqs_dbg64_read(c, 16)
st = max(1, c[2])
it = max(1, c[6])
print("softmax per step: wait-for-S %.0f  S->P %.0f  steps %d"
      % (c[0] / st, c[1] / st, st))
print("mma per kv-iter: wait-for-P %.0f  wait-for-K/V %.0f  total %.0f  iters %d"
      % (c[4] / it, c[7] / it, c[5] / it, it))

"""Cycle accounting of the CTA-pair kernel (or, with --d64, the 1-CTA D=64 kernel: counters 0-2 and
4-6 only) (debug build with -DCQS_DBG_TIMING, loaded via CQS_LIB).
Counters: 0 softmax wait-for-S cycles, 1 softmax S->P cycles, 2 softmax tile count,
4 MMA wait-for-P cycles, 5 MMA warp total cycles, 6 MMA kv-iterations."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cqs_synth
import paper_2604_20819_b200 as cqs

L = cqs.lib()
D = 64 if "--d64" in sys.argv else 128
q, k, v = cqs_synth.torch_qkv(1, 32, 131072, D, 20260418, dtype=torch.bfloat16, device="cuda")
cqs.attention(q, k, v, depth=1)
torch.cuda.synchronize()
rd, rs = (L.cqs_dbg1_read, L.cqs_dbg1_reset) if D == 64 else (L.cqs_dbg_read, L.cqs_dbg_reset)
rs()
cqs.attention(q, k, v, depth=1)
torch.cuda.synchronize()
c = (ctypes.c_ulonglong * 16)()
rd(c, 16)
tiles = max(1, c[2])
print("softmax: wait-for-S %.0f cyc/tile, S->P %.0f cyc/tile, tiles %d" % (c[0] / tiles, c[1] / tiles, tiles))
print("softmax phases per tile: LDTM %.0f  max+rescale %.0f  gate %.0f  exp %.0f  sum/pack/STTM/arrive %.0f" % tuple(c[i] / tiles for i in range(7, 12)))
print("mma: wait-for-V-tile %.0f cyc/kv-iter" % (c[3] / max(1, c[6])))
print("mma: wait-for-P %.0f cyc/tile-iter, total %.0f cyc/kv-iter (per pair), iters %d" % (
    c[4] / max(1, c[6]) / 2, c[5] / max(1, c[6]), c[6]))

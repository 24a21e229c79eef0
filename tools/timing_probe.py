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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cqs.attention(q, k, v, depth=1)
e1.record()
torch.cuda.synchronize()
wall_ms = e0.elapsed_time(e1)
c = (ctypes.c_ulonglong * 32)()
rd(c, 32 if D == 128 else 16)
tiles = max(1, c[2])
print("softmax: wait-for-S %.0f cyc/tile, S->P %.0f cyc/tile, tiles %d" % (c[0] / tiles, c[1] / tiles, tiles))
print("softmax phases per tile: LDTM %.0f  max+rescale %.0f  gate %.0f  exp %.0f  sum/pack/STTM/arrive %.0f" % tuple(c[i] / tiles for i in range(7, 12)))
print("mma: wait-for-V-tile %.0f cyc/kv-iter" % (c[3] / max(1, c[6])))
print("mma: wait-for-P %.0f cyc/tile-iter, total %.0f cyc/kv-iter (per pair), iters %d" % (
    c[4] / max(1, c[6]) / 2, c[5] / max(1, c[6]), c[6]))
if D == 128 and c[14]:
    ctas = c[14]
    print("cta lifetime: %.0f cycles, %.1f us avg; in-kernel clock %.0f MHz; CTAs %d; "
          "SM occupancy by attention CTAs %.3f of %d SMs x %.2f ms; epilogue %.0f cyc/warp-tile" % (
              c[12] / ctas, c[13] / ctas / 1e3, c[12] / c[13] * 1e3, ctas,
              c[13] / 1e6 / (148 * wall_ms), 148, wall_ms, c[3] / max(1, ctas * 8)))
    # per-SM view: steady-state loop cycles per kv-iter vs whole-lifetime cycles per kv-iter
    print("lifetime cycles per kv-iter (per CTA) %.0f" % (c[12] / ctas / (c[6] / (ctas / 2))))
if D == 128 and c[19]:
    n = c[19]
    print("warp 4 (tile 0, sub 0) per CTA: loop starts %.0f cyc after entry, loop %.0f cyc, "
          "epilogue ends %.0f cyc after entry" % (c[16] / n, c[17] / n, c[18] / n))

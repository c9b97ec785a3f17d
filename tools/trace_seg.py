"""Per-segment (accumulator-stage) timeline of CTAs 0..7 (debug build
-DLQG_TRACE_SEG -> liblqg_traceseg.so, BF16 output kernel): when the MMA warp
started waiting for a stage, got it, issued the segment's last MMA, and when
the epilogue saw the accumulator, released the stage and finished the segment
(us from the first event). Shows whether the MMA waits on the epilogue and
how long each epilogue segment takes under load.

  python tools/trace_seg.py 8192x8192x4096 [cta=0] [knob=v ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_01229_b200 import _lib

_lib.LIB_PATH = os.path.join(_lib.HERE, os.environ.get("TRACE_LIB", "liblqg_traceseg.so"))
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

n, k, m = map(int, sys.argv[1].split("x"))
ctas = [0]
for kv in sys.argv[2:]:
    kk, v = kv.split("=")
    if kk == "cta":
        ctas = [int(c) for c in v.split(",")]
    else:
        lqg.tune_set(kk, int(v))
dw = lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128)
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    dw.gemm(q, ts, out=y)
torch.cuda.synchronize()
buf = np.zeros(8 * 32 * 16, np.int64)
ctypes.CDLL(_lib.LIB_PATH).lqg_debug_seg_kind3(buf.ctypes.data_as(ctypes.c_void_p))
ev = buf.reshape(8, 32, 16)
t0 = ev[:, :, :6][ev[:, :, :6] > 0].min()
kinds = {0: "whole", 1: "contrib", 2: "finish"}
for cta in ctas:
    print(f"{sys.argv[1]}: CTA {cta} (us from the first event)")
    print("  seg   kind  kbs  mma-wait  stage-ok  last-mma  epi-acc  released  epi-done   acc-wait  epi-len"
          "  ld-cyc  st-cyc")
    tot_wait = 0.0
    for j in range(32):
        r = ev[cta, j]
        if not r[3] and not r[1]:
            break
        f = lambda v: (v - t0) / 1e3 if v else float("nan")
        wait = (r[1] - r[0]) / 1e3 if r[0] and r[1] else float("nan")
        tot_wait += wait if wait == wait else 0.0
        epi = (r[5] - r[3]) / 1e3 if r[3] and r[5] else float("nan")
        print(f"  {j:3d} {kinds.get(int(r[7]), '?'):>7s} {int(r[6]):4d} {f(r[0]):9.2f} {f(r[1]):9.2f} {f(r[2]):9.2f}"
              f" {f(r[3]):8.2f} {f(r[4]):9.2f} {f(r[5]):9.2f} {wait:9.2f} {epi:8.2f} {int(r[8]):7d} {int(r[9]):7d}")
    print(f"  total MMA acc-wait {tot_wait:.2f} us")

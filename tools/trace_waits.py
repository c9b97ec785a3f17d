"""Per-role wait breakdown of one GEMM launch (trace build, -DLQG_TRACE):
dequant warpgroup 0 waiting for weight chunks / TMEM A slots, and the MMA
warp waiting for the accumulator stage / A operand / activation tile, as
fractions of each role's loop cycles (median over CTAs).

  python tools/trace_waits.py 28672x8192x128 [knob=value ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_01229_b200 import _lib

_lib.LIB_PATH = os.path.join(_lib.HERE, os.environ.get("TRACE_LIB", "liblqg_trace.so"))
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

n, k, m = map(int, sys.argv[1].split("x"))
for kv in sys.argv[2:]:
    kk, v = kv.split("=")
    lqg.tune_set(kk, int(v))
w = torch.randn(n, k, device="cuda") * 0.02
dw = lqg.DeviceWeights.quantize(w, 128)
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    dw.gemm(q, ts, out=y)
torch.cuda.synchronize()
L = _lib.lib()
buf = np.zeros(8 * 160 * 16, np.uint64)
L.lqg_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
allr = buf.reshape(8, 160, 16).astype(np.int64)
last = max(range(8), key=lambda sl: allr[sl][:, 0].max())
r = allr[last]
dq = r[r[:, 11] > 0]
mm = r[r[:, 15] > 0]
span = (r[:, :9].max() - r[r[:, 0] > 0, 0].min()) / 1e3
print(f"{sys.argv[1]} {' '.join(sys.argv[2:])}: {len(mm)} MMA CTAs, launch span {span:.1f} us")
print(f"  dequant WG0: wait W {np.median(dq[:, 9] / dq[:, 11]) * 100:5.1f}%  "
      f"wait A-slot {np.median(dq[:, 10] / dq[:, 11]) * 100:5.1f}%  loop cycles {np.median(dq[:, 11]):.0f}")
for j, nm in ((12, "wait acc"), (13, "wait A (dequant)"), (14, "wait X tile"), (3, "issue block")):
    frac = mm[:, j] / mm[:, 15]
    print(f"  MMA {nm:18s} median {np.median(frac) * 100:5.1f}%  max {frac.max() * 100:5.1f}%")
print(f"  MMA loop cycles median {np.median(mm[:, 15]):.0f}")
# timeline (us from the first CTA's entry): entry, prologue done, X producer
# past griddepcontrol.wait, first MMA, last MMA, epilogue's last accumulator
t0 = r[r[:, 0] > 0, 0].min()
for j, nm in ((0, "entry"), (1, "prologue done"), (2, "X after PDL wait"), (4, "first MMA"), (5, "last MMA"),
              (6, "last acc ready")):
    v = r[r[:, j] > 0, j]
    if len(v):
        q = np.percentile((v - t0) / 1e3, [0, 50, 100])
        print(f"  {nm:18s} min {q[0]:6.2f}  med {q[1]:6.2f}  max {q[2]:6.2f} us")

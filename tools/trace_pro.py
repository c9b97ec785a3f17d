"""Prologue breakdown of one launch (build with -DLQG_TRACE -DLQG_TRACE_PRO into
liblqg_tracepro.so): entry, barriers initialised, TMEM allocated, first
__syncthreads, prologue done, X producer past griddepcontrol.wait, first / last
MMA, last accumulator ready; plus the SM of every CTA (placement check).

  python tools/trace_pro.py 4096x4096x16 [launches=3]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_01229_b200 import _lib

_lib.LIB_PATH = os.path.join(_lib.HERE, "liblqg_tracepro.so")
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

n, k, m = map(int, sys.argv[1].split("x"))
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = torch.randn(n, k, device="cuda") * 0.02
dw = lqg.DeviceWeights.quantize(w, 128)
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
for _ in range(R):
    dw.gemm(q, ts, out=y)
torch.cuda.synchronize()
buf = np.zeros(8 * 160 * 16, np.uint64)
_lib.lib().lqg_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
allr = buf.reshape(8, 160, 16).astype(np.int64)
last = max(range(8), key=lambda sl: allr[sl][:, 0].max())
r = allr[last]
used = r[:, 0] > 0
r = r[used]
t0 = r[:, 0].min()
print(f"{sys.argv[1]}: {used.sum()} CTAs on {len(set(r[:, 3].tolist()))} distinct SMs (us from first entry)")
for j, nm in ((0, "entry"), (9, "barriers init"), (10, "TMEM allocated"), (11, "first syncthreads"),
              (1, "prologue done"), (2, "X past PDL wait"), (4, "first MMA"), (5, "last MMA"),
              (6, "last acc ready")):
    v = r[r[:, j] > 0, j]
    if len(v):
        qq = np.percentile((v - t0) / 1e3, [0, 50, 100])
        print(f"  {nm:18s} min {qq[0]:6.2f}  med {qq[1]:6.2f}  max {qq[2]:6.2f} us")

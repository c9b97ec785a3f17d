"""MMA-warp wait breakdown per CTA (trace build): cycles waiting for the
accumulator stage, the A operand (dequant), the activation tile, and total."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_01229_b200 import _lib
_lib.LIB_PATH = os.path.join(_lib.HERE, "liblqg_trace.so")
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg
n, k, m = map(int, sys.argv[1].split("x"))
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
full = r.copy()
tot = r[:, 15]
used = tot > 0
r = r[used]
dq = full[full[:, 11] > 0]
for who, rows in (("all", dq), ("leaders", dq[0::2]), ("peers", dq[1::2])):
    print(f"  dequant ({who}): wait W {np.median(dq[:,2]/dq[:,11])*100 if who=='all' else np.median(rows[:,2]/rows[:,11])*100:5.1f}%  "
          f"wait A-slot {np.median(rows[:,3]/rows[:,11])*100:5.1f}%  "
          f"tmem_st_wait {np.median(rows[:,4]/rows[:,11])*100:5.1f}%  arrive {np.median(rows[:,5]/rows[:,11])*100:5.1f}%")
print(f"{sys.argv[1]} pair={os.environ.get('LQG_PAIR','0')}: MMA-issuing CTAs {used.sum()}")
for j, nm in ((12, "wait acc"), (13, "wait A (dequant)"), (14, "wait X tile")):
    frac = r[:, j] / r[:, 15]
    print(f"  {nm:18s} median {np.median(frac)*100:5.1f}%  max {frac.max()*100:5.1f}%")
print(f"  total MMA-loop cycles median {np.median(r[:,15]):.0f}")

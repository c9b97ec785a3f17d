"""Per-CTA timeline of one GEMM launch (debug build with -DLQG_TRACE)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_01229_b200 import _lib
_lib.LIB_PATH = os.path.join(_lib.HERE, "liblqg_trace.so")
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

NAMES = ["entry", "prologue", "griddep", "dq_first_w", "mma_first", "mma_last", "epi_last_acc", "epi_end", "exit", "contrib_pub", "fin_spun"]
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
allr = buf.reshape(8, 160, 16)
last = max(range(8), key=lambda sl: allr[sl][:, 0].max())  # the most recent launch
raw = allr[last].copy()
t = raw[:, :11].astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
print(f"{n}x{k}x{m}: CTAs={used.sum()}  (us relative to first CTA entry)")
for j, nm in enumerate(NAMES):
    c = rel[:, j]
    c = c[t[:, j] > 0]
    if len(c):
        print(f"  {nm:14s} min {c.min():7.2f}  med {np.median(c):7.2f}  max {c.max():7.2f}")

# slowest CTAs: their split roles
order = np.argsort(-rel[:, 7])
import sys as _s
for i in order[:int(_s.argv[2]) if len(_s.argv) > 2 else 2]:
    cf, ce = int(raw[i, 11]) >> 32, int(raw[i, 11]) & 0xFFFFFFFF
    print(f"  cta {i}: last_acc {rel[i,6]:.2f} epi_end {rel[i,7]:.2f} contrib_pub {rel[i,9] if t[i,9] else -1:.2f} "
          f"fin_spun {rel[i,10] if t[i,10] else -1:.2f} first_loads {(int(raw[i,12]) - t0)/1000 if raw[i,12] else -1:.2f} spins {int(raw[i,13])} contributors [{cf},{ce})"
          + "".join(f" | c{c}: pub {rel[c,9]:.2f} last_acc {rel[c,6]:.2f}" for c in range(cf, ce) if c < len(rel)))

"""Per-k-block timeline of CTA 0 (debug build -DLQG_TRACE_KB -> liblqg_tracekb.so,
BF16 output kernel): when each k-block's weight chunk and activation tile were
requested, when its dequant warpgroup saw the weights, got the TMEM A slot and
published it, and when the MMA warp saw the A operand and issued (cycles,
relative to the first event shown).

  python tools/trace_kb.py 8192x8192x4096 [first_kb=16] [count=24] [knob=v ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_01229_b200 import _lib

_lib.LIB_PATH = os.path.join(_lib.HERE, os.environ.get("TRACE_LIB", "liblqg_tracekb.so"))
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

n, k, m = map(int, sys.argv[1].split("x"))
first = int(sys.argv[2]) if len(sys.argv) > 2 and "=" not in sys.argv[2] else 16
count = int(sys.argv[3]) if len(sys.argv) > 3 and "=" not in sys.argv[3] else 24
for kv in sys.argv[2:]:
    if "=" in kv:
        kk, v = kv.split("=")
        lqg.tune_set(kk, int(v))
dw = lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128)
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    dw.gemm(q, ts, out=y)
torch.cuda.synchronize()
buf = np.zeros(2 * 64 * 8, np.int64)
C = ctypes.CDLL(_lib.LIB_PATH)
C.lqg_debug_kb_kind3(buf.ctypes.data_as(ctypes.c_void_p))
both = buf.reshape(2, 64, 8)
cta = int(os.environ.get("CTA", "0"))  # 0: CTA 0 (a pair's leader), 1: CTA 1 (its peer)
ev = both[cta]
names = ["W req", "X req", "dq W ok", "dq A free", "dq A pub", "mma A ok", "mma issued", "dq st done"]
sel = ev[first:first + count, :8]
allsel = both[:, first:first + count, :8]
t0 = allsel[allsel > 0].min()  # one global clock (%globaltimer, ns) for both CTAs
print(f"{sys.argv[1]}: CTA {cta}, k-blocks {first}..{first + count - 1} (ns from the first event of either CTA)")
print("  kb " + "".join(f"{nm:>11s}" for nm in names) + "   A-pub->mma-ok  issue->next-A-ok")
for r, row in enumerate(sel):
    i = first + r
    vals = "".join(f"{(v - t0) if v else -1:11d}" for v in row)
    lag = row[5] - row[4] if row[4] and row[5] else -1
    nxt = ev[i + 1, 5] - row[6] if i + 1 < 64 and ev[i + 1, 5] and row[6] else -1
    print(f"  {i:2d} {vals}   {lag:8d}   {nxt:8d}")
d = np.diff(ev[first:first + count, 6])
print(f"  MMA issue period: median {np.median(d):.0f} ns/k-block")

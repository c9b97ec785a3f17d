"""Timeline of a chain of back-to-back launches inside a CUDA graph (PDL
edges, as in bench.py), from the LQG_TRACE_PRO build (liblqg_tracepro.so):
per launch, its CTAs' entry, griddepcontrol.wait release (X producer), first
and last MMA, last accumulator ready and CTA exit, in us from the first entry
of the window. Shows whether consecutive launches overlap (co-resident CTAs
prefill their rings while the previous grid runs).

  python tools/trace_chain.py 4096x4096x16 [copies=16] [knob=value ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_01229_b200 import _lib

_lib.LIB_PATH = os.path.join(_lib.HERE, os.environ.get("LQG_TRACE_LIB", "liblqg_tracepro.so"))
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

n, k, m = map(int, sys.argv[1].split("x"))
copies = 16
for kv in sys.argv[2:]:
    kk, v = kv.split("=")
    if kk == "copies":
        copies = int(v)
    else:
        lqg.tune_set(kk, int(v))
dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128) for _ in range(copies)]
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
ws = lqg.Workspace(0)
while lqg.launch_count() % 8:  # align trace slots with the graph's launch order
    dws[0].gemm(q, ts, out=y, workspace=ws)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
    for dw in dws:
        dw.gemm(q, ts, out=y, workspace=ws)
torch.cuda.current_stream().wait_stream(st)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"{sys.argv[1]} {' '.join(sys.argv[2:])}: {copies} launches in {e0.elapsed_time(e1) * 1e3:.1f} us "
      f"= {e0.elapsed_time(e1) * 1e3 / copies:.2f} us/launch")
buf = np.zeros(8 * 160 * 16, np.uint64)
_lib.lib().lqg_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
allr = buf.reshape(8, 160, 16).astype(np.int64)
live = [sl for sl in range(8) if (allr[sl][:, 0] > 0).any()]
order = sorted(live, key=lambda sl: allr[sl][allr[sl][:, 0] > 0, 0].min())
t0 = min(allr[sl][allr[sl][:, 0] > 0, 0].min() for sl in live)
print("  launch:   entry[min,max]   PDL-rel   MMA[first,last]  acc[med,max] pub-max  epi-done[med,max]  exit[min,max]  (us)")
for sl in order:
    r = allr[sl]
    r = r[r[:, 0] > 0]
    f = lambda j, fn: (fn(r[r[:, j] > 0, j]) - t0) / 1e3 if (r[:, j] > 0).any() else float("nan")
    print(f"  slot {sl}: {f(0, np.min):6.2f} {f(0, np.max):6.2f}  {f(2, np.median):7.2f}  "
          f"{f(4, np.median):6.2f} {f(5, np.max):6.2f}  {f(6, np.median):6.2f} {f(6, np.max):6.2f} {f(7, np.max):6.2f}  "
          f"{f(13, np.median):6.2f} {f(13, np.max):6.2f}  {f(12, np.min):6.2f} {f(12, np.max):6.2f}"
          f" | fin: start {f(9, np.median):6.2f} flags {f(10, np.median):6.2f}/{f(10, np.max):6.2f}"
          f" gather {f(11, np.median):6.2f} ch0-summed {f(8, np.median):6.2f} ch0-stored {f(15, np.median):6.2f}"
          f" stored {f(14, np.median):6.2f}/{f(14, np.max):6.2f}"
          f"   SMs {len(set(r[:, 3].tolist()))}")

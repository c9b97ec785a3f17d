"""Per-SM timelines of the 70B 4-layer decode step under the dynamic
(work-stealing) schedule (debug build -DLQG_TRACE, liblqg_trace.so).
  python tools/trace_dyn.py [M]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_01229_b200 import _lib
_lib.LIB_PATH = os.environ.get("LQG_LIB_PATH", os.path.join(_lib.HERE, "liblqg_trace.so"))
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

EV = ["entry", "prologue", "griddep", "mma_first", "mma_last", "epi_end", "exit"]
ACC = {8: "claim_wait_us", 9: "units", 10: "uidpush_wait_us", 11: "mma_accwait_us", 12: "prod_emptywait_us", 13: "mma_afull_wait_us", 14: "mma_xfull_wait_us"}
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
shapes = [(10240, 8192), (8192, 8192), (28672, 8192), (8192, 28672)]
g = torch.Generator(device="cuda"); g.manual_seed(1)
layers = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128) for n, k in shapes]
xs = {k: lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda")) for k in (8192, 28672)}
ys = [torch.empty(m, n, dtype=torch.bfloat16, device="cuda") for n, _ in shapes]
ws = lqg.Workspace(0)
L = _lib.lib()


def step():
    for (n, k), dw, y in zip(shapes, layers, ys):
        q, ts = xs[k]
        dw.gemm(q, ts, out=y, workspace=ws)


step(); torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
    step(); step()
torch.cuda.current_stream().wait_stream(s)
for _ in range(5):
    gr.replay()
torch.cuda.synchronize()
buf = np.zeros(8 * 160 * 16, np.uint64)
L.lqg_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
raw = buf.reshape(8, 160, 16).astype(np.int64)
live = [sl for sl in range(8) if (raw[sl][:, 0] > 0).any()]
first = {sl: raw[sl][raw[sl][:, 0] > 0, 0].min() for sl in live}
slots = sorted(live, key=lambda sl: first[sl])[-4:]
t0 = first[slots[0]]
print(f"M={m}: us relative to the first CTA entry of layer 0 (min/med/max over SMs)")
for li, sl in enumerate(slots):
    t = raw[sl]
    t = t[t[:, 0] > 0]
    n, k = shapes[li]
    print(f" layer {li} ({n}x{k}) SMs={len(t)}")
    for j, nm in enumerate(EV):
        c = t[:, j]
        c = (c[c > 0] - t0) / 1000.0
        if len(c):
            print(f"   {nm:13s} {c.min():8.2f} {np.median(c):8.2f} {c.max():8.2f}")
    for j, nm in ACC.items():
        c = t[:, j] / (1 if j == 9 else 1000.0)
        print(f"   {nm:17s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f} sum {c.sum():8.1f}")

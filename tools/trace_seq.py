"""Per-GEMM timelines of the 70B 4-layer decode step (debug build -DLQG_TRACE).
  python tools/trace_seq.py [M]      (env knobs of liblqg apply, e.g. LQG_PDL_TRIGGER)
Replays the step as a CUDA graph and prints each launch's event spread
(min/med/max over CTAs) on one global clock."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_01229_b200 import _lib
_lib.LIB_PATH = os.environ.get("LQG_LIB_PATH", os.path.join(_lib.HERE, "liblqg_trace.so"))
_lib._stale = lambda: False
import paper_2509_01229_b200 as lqg

NAMES = ["entry", "prologue", "griddep", "dq_first_w", "mma_first", "mma_last", "epi_last_acc", "epi_end", "exit"]
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
base = L.lqg_kernel_launch_count()
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
# the last four launches by start time = the second step of the last replay
live = [sl for sl in range(8) if (raw[sl][:, 0] > 0).any()]
first = {sl: raw[sl][raw[sl][:, 0] > 0, 0].min() for sl in live}
slots = sorted(live, key=lambda sl: first[sl])[-4:]
t0 = first[slots[0]]
print(f"M={m}: us relative to the first CTA entry of layer 0 (min/med/max over CTAs)")
for li, sl in enumerate(slots):
    t = raw[sl]
    t = t[t[:, 0] > 0]
    n, k = shapes[li]
    print(f" layer {li} ({n}x{k}) CTAs={len(t)}")
    for j, nm in enumerate(NAMES):
        c = t[:, j]
        c = (c[c > 0] - t0) / 1000.0
        if len(c):
            print(f"   {nm:13s} {c.min():8.2f} {np.median(c):8.2f} {c.max():8.2f}")

# slowest CTAs of each layer: start, mainloop, split role
for li, sl in enumerate(slots):
    t = raw[sl]
    rel = (t[:, :11] - t0) / 1000.0
    order = np.argsort(-t[:, 7])
    print(f" layer {li} slowest:")
    for i in order[:4]:
        cf, ce = int(t[i, 11]) >> 32, int(t[i, 11]) & 0xFFFFFFFF
        fl = (int(t[i, 12]) - t0) / 1000.0 if t[i, 12] else -1
        print(f"   cta {i:3d}: entry {rel[i,0]:6.2f} gd {rel[i,2]:6.2f} mma {rel[i,4]:6.2f}..{rel[i,5]:6.2f} "
              f"acc {rel[i,6]:6.2f} end {rel[i,7]:6.2f} pub {rel[i,9] if t[i,9] else -1:6.2f} fin_first {fl:6.2f} "
              f"spins {int(t[i,13])} contrib [{cf},{ce})"
              + "".join(f" | c{c}: entry {rel[c,0]:.2f} pub {rel[c,9]:.2f}" for c in range(cf, ce) if c < len(rel)))

# lateness vs blockIdx: median (over buckets of 16 CTAs) of entry and mma_last
print(" entry / mma_last / exit by blockIdx bucket of 16 (us):")
for li, sl in enumerate(slots):
    t = raw[sl]
    rel = (t[:, :11] - t0) / 1000.0
    row = []
    for b in range(0, 148, 16):
        r = rel[b:min(b + 16, 148)]
        row.append(f"{np.median(r[:,0]):5.1f}/{np.median(r[:,5]):5.1f}/{np.median(r[:,8]):5.1f}")
    print(f"  layer {li}: " + " ".join(row))

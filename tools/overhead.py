"""Decompose the fixed per-launch cost: graph-replayed empty kernel vs tiny GEMMs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_01229_b200 as lqg


def graph_time(fn, R=50):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(R):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R * 1e3


x = torch.zeros(1, device="cuda")
print(f"empty torch kernel (x.add_): {graph_time(lambda: x.add_(1)):.2f} us")
for (n, k, m) in [(128, 256, 16), (128 * 148, 256, 16), (128, 256 * 148, 16), (128 * 74, 512, 16),
                  (8192, 256, 16), (4096, 4096, 16), (8192, 28672, 16)]:
    w = torch.randn(n, k, device="cuda") * 0.02
    dw = lqg.DeviceWeights.quantize(w, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    t = graph_time(lambda: dw.gemm(q, ts, out=y))
    print(f"n={n} k={k} m={m}: {t:.2f} us")

# eager host cost per call (python wrapper + C ABI launch), and the C ABI alone
import time
from paper_2509_01229_b200 import _lib
n, k, m = 4096, 11008, 16
w = torch.randn(n, k, device="cuda") * 0.02
dw = lqg.DeviceWeights.quantize(w, 128)
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
ws = lqg.Workspace(0)
for _ in range(10):
    dw.gemm(q, ts, out=y, workspace=ws)
torch.cuda.synchronize()
R = 200
t0 = time.perf_counter()
for _ in range(R):
    dw.gemm(q, ts, out=y, workspace=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"eager python gemm(): host {1e6 * (t1 - t0) / R:.2f} us/call, wall incl. drain {1e6 * (t2 - t0) / R:.2f} us/call")
L = _lib.lib()
args = (dw.handle, q.data_ptr(), q.stride(0), ts.data_ptr(), m, y.data_ptr(), y.stride(0), 3, ws.handle, None)
t0 = time.perf_counter()
for _ in range(R):
    L.lqg_gemm_w4a8(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"eager C ABI lqg_gemm_w4a8: host {1e6 * (t1 - t0) / R:.2f} us/call, wall {1e6 * (t2 - t0) / R:.2f} us/call")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize()
e0.record(); L.lqg_gemm_w4a8(*args); e1.record(); torch.cuda.synchronize()
print(f"one eager C ABI call between events: {e0.elapsed_time(e1) * 1e3:.2f} us")
e0.record(); dw.gemm(q, ts, out=y, workspace=ws); e1.record(); torch.cuda.synchronize()
print(f"one eager python call between events: {e0.elapsed_time(e1) * 1e3:.2f} us")

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

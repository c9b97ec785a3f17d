"""Epilogue cost in isolation: a one-k-block GEMM (K = 256) with many tokens
is all epilogue (scale, cast, store) -- device time per output element for
each output kind, graph of R launches.

  python tools/epi_cost.py [--n 8192] [--m 4096]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--k", type=int, default=256)
a = ap.parse_args()
dw = lqg.DeviceWeights.quantize(torch.randn(a.n, a.k, device="cuda") * 0.02, 128)
q, ts = lqg.quantize_activations(torch.randn(a.m, a.k, device="cuda"))
for name, dt in (("int32", None), ("f32", torch.float32), ("bf16", torch.bfloat16)):
    y = torch.empty(a.m, a.n, dtype=dt or torch.int32, device="cuda")
    run = (lambda: dw.gemm_accum(q, out=y)) if dt is None else (lambda: dw.gemm(q, ts, out=y))
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(10):
            run()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    outs = a.m * a.n
    print(f"{name:6s} n={a.n} k={a.k} m={a.m}: {t * 1e6:8.1f} us  {outs / t / 1e9:8.1f} Gout/s  "
          f"{outs * y.element_size() / t / 1e9:7.1f} GB/s written  {t * 1.9e9 * 148 / outs * 128:7.1f} SM-cycles per 128 outputs")

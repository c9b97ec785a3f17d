"""Per-shape device time vs persistent grid size (tune knob `grid`), graph of
R launches rotating over 3 weight copies:

  python tools/grid_sweep.py [--ms 16,128] [--workload llama2-70b|llama2-7b] [--grids 0,64,96,128]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="16,128")
ap.add_argument("--workload", default="llama2-70b")
ap.add_argument("--grids", default="0,64,80,96,112,128")
a = ap.parse_args()


def tgraph(fn, R=12):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(R):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / R * 1e3)
    return best


grids = [int(x) for x in a.grids.split(",")]
for name, n, k in WORKLOADS[a.workload]["shapes"]:
    dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128) for _ in range(3)]
    for m in [int(x) for x in a.ms.split(",")]:
        q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
        y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        it = [0]

        def fn():
            dws[it[0] % 3].gemm(q, ts, out=y)
            it[0] += 1
        res = {}
        for grid in grids:
            lqg.tune_set("grid", grid)
            res[grid] = tgraph(fn)
        lqg.tune_set("grid", 0)
        print(f"{name:8s} m={m:4d} " + " ".join(f"g{g}={t:6.1f}" for g, t in res.items()), flush=True)

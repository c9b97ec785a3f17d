"""Per-shape device time under schedule-knob variants (token-tile cap, CTA-pair
policy, quad mode, grid), graph of R launches rotating over 3 weight copies so
the weights stream from HBM. Every variant is bit-exact (the knobs only move
the schedule); this finds where the default rules leave time on the table:

  python tools/sched_sweep.py [--workload llama2-7b] [--ms 256,512,1024]
      [--variants "default;max_bn=128;pair=0;max_bn=96,pair=0"]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="128,256,512,1024")
ap.add_argument("--workload", default="llama2-7b")
ap.add_argument("--variants", default="default;max_bn=128;max_bn=160;max_bn=96;pair=0;max_bn=128,pair=0;no_quad=1")
ap.add_argument("--json", default="")
a = ap.parse_args()

KNOBS = ("max_bn", "pair", "pair_min_m", "grid", "no_quad", "no_dp", "raster_gm", "auto_tile")


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
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / R * 1e3)
    return sorted(ts)[len(ts) // 2]


def parse(v):
    if v == "default":
        return {}
    return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in v.split(",")}


variants = [(v, parse(v)) for v in a.variants.split(";")]
DEFAULTS = {kk: lqg.tune_get(kk) for kk in KNOBS}
rows = []
for name, n, k in WORKLOADS[a.workload]["shapes"]:
    dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128) for _ in range(3)]
    for m in [int(x) for x in a.ms.split(",")]:
        q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
        y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        ref = None
        it = [0]

        def fn():
            dws[it[0] % 3].gemm(q, ts, out=y)
            it[0] += 1
        res = {}
        for vname, knobs in variants:
            for kk, vv in DEFAULTS.items():
                lqg.tune_set(kk, vv)
            for kk, vv in knobs.items():
                lqg.tune_set(kk, vv)
            dws[0].gemm(q, ts, out=y)
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            elif not torch.equal(ref, y):
                raise SystemExit(f"{name} m={m} {vname}: output differs from the default schedule")
            res[vname] = tgraph(fn)
        for kk, vv in DEFAULTS.items():
            lqg.tune_set(kk, vv)
        best = min(res, key=res.get)
        rows.append({"shape": name, "n": n, "k": k, "m": m, "us": res, "best": best})
        print(f"{name:8s} m={m:5d} " + " ".join(f"{v}={t:6.1f}" for v, t in res.items()) + f"  best={best}",
              flush=True)
if a.json:
    with open(a.json, "w") as f:
        json.dump(rows, f, indent=1)

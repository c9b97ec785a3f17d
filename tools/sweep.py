"""Per-M device time of a workload's layer GEMMs (CUDA graph of R rotations of
the layer GEMMs per M; weights > L2), optionally under launch-schedule knobs.

  python tools/sweep.py --workload llama2-70b --ms 1,16,64,128,256,1024,4096 \
      [--tune x_ring_bytes=32768,pair=1] [--per-shape]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_2509_01229_b200 as lqg
from bench import WORKLOADS, algo_bytes, algo_ops, load_peaks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama2-70b")
    ap.add_argument("--ms", default="1,16,64,128,256,1024,4096")
    ap.add_argument("--tune", default="")
    ap.add_argument("--per-shape", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for kv in filter(None, a.tune.split(",")):
        k, v = kv.split("=")
        lqg.tune_set(k, int(v))
    wl = WORKLOADS[a.workload]
    ms = [int(x) for x in a.ms.split(",")]
    peaks = load_peaks()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    layers = []
    for name, n, k in wl["shapes"]:
        w = torch.randn(n, k, generator=g, device=dev) * 0.02
        layers.append((name, n, k, lqg.DeviceWeights.quantize(w, 128)))
        del w
    xs = {}
    for k in {k for _, _, k in wl["shapes"]}:
        xs[k] = lqg.quantize_activations(torch.randn(max(ms), k, generator=g, device=dev))
    ys = {name: torch.empty(max(ms), n, dtype=torch.bfloat16, device=dev) for name, n, _, _ in layers}
    ws = lqg.Workspace(0)

    def timed(fn, R=3):
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st), torch.cuda.graph(gr, stream=st):
            for _ in range(R):
                fn()
        torch.cuda.current_stream().wait_stream(st)
        gr.replay()
        torch.cuda.synchronize()
        samples = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(a.reps):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1) * 1e-3 / (a.reps * R))
        return statistics.median(samples)

    for m in ms:
        def step(sel=None):
            for name, n, k, dw in layers:
                if sel is None or name == sel:
                    q, ts = xs[k]
                    dw.gemm(q[:m], ts[:m], out=ys[name][:m], workspace=ws)
        if m <= 64:
            time.sleep(1.0)
        t = timed(step)
        ops = sum(algo_ops(m, n, k) for _, n, k, _ in layers)
        byts = sum(algo_bytes(m, n, k) for _, n, k, _ in layers)
        print(f"M={m:5d} step {t*1e6:8.1f} us  {ops/t/1e12:7.1f} TOPS  hbm {byts/t/1e9/peaks['hbm_gbs']:.3f}  "
              f"int8(2xbf16) {ops/t/1e12/(2*1686.1):.3f}", flush=True)
        if a.per_shape:
            for name, n, k, _ in layers:
                ts_ = timed(lambda: step(name), R=4 if n * k < 120e6 else 3)
                print(f"     {name:8s} {n}x{k}: {ts_*1e6:7.1f} us  hbm {algo_bytes(m, n, k)/ts_/1e9/peaks['hbm_gbs']:.3f}"
                      f"  tops {algo_ops(m, n, k)/ts_/1e12:.0f}", flush=True)


if __name__ == "__main__":
    main()

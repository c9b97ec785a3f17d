"""Launch one W4A8 GEMM shape a few times (for ncu captures).

  ncu --set full --clock-control none --import-source on -k regex:lqg_w4a8 -s 2 -c 1 \
      -o gpurun_out/prof_down_m16 python tools/profile_one.py --n 8192 --k 28672 --m 16
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2509_01229_b200 as lqg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=28672)
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--g", type=int, default=128)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--tune", action="append", default=[], help="knob=value (repeatable)")
    a = ap.parse_args()
    for kv in a.tune:
        kk, vv = kv.split("=")
        lqg.tune_set(kk, int(vv))
    torch.manual_seed(0)
    w = torch.randn(a.n, a.k, device="cuda") * 0.02
    dw = lqg.DeviceWeights.quantize(w, a.g)
    del w
    x = torch.randn(a.m, a.k, device="cuda")
    q, ts = lqg.quantize_activations(x)
    y = torch.empty(a.m, a.n, dtype=torch.bfloat16, device="cuda")
    for _ in range(a.iters):
        dw.gemm(q, ts, out=y)
    torch.cuda.synchronize()
    if a.time:
        # CUDA graph of R launches: device time without host launch gaps.
        # Weights rotate over 4 copies when they would fit in L2.
        copies = [dw]
        if a.n * a.k // 2 < 200 * 2**20:
            for i in range(3):
                w = torch.randn(a.n, a.k, device="cuda") * 0.02
                copies.append(lqg.DeviceWeights.quantize(w, a.g))
                del w
        R = 20
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            for r in range(R):
                copies[r % len(copies)].gemm(q, ts, out=y)
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / R * 1e-3
        byts = a.n * a.k // 2 + 2 * a.n * a.k // a.g + 4 * a.n + a.m * a.k + 4 * a.m + 2 * a.m * a.n
        print(f"n={a.n} k={a.k} m={a.m}: {t*1e6:.1f} us  {byts/t/1e9:.0f} GB/s  "
              f"{2*a.m*a.n*a.k/t/1e12:.1f} TOPS")


if __name__ == "__main__":
    main()

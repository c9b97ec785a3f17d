"""Why does the same M = 4096 LLaMA-2-70B 4-GEMM step time differently in
bench.py and tools/ab.py? Times the step (CUDA graph, 3 rotations) for two
activation distributions (plain randn vs bench.py's 0.1 % x20 outliers) right
after idle and after ~8 s of continuous tensor work, with SM clock and power
sampled by NVML during each timing."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch

import paper_2509_01229_b200 as lqg

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
shapes = [(10240, 8192), (8192, 8192), (28672, 8192), (8192, 28672)]
M = int(os.environ.get("M", "4096"))
g = torch.Generator(device="cuda")
layers = []
for li, (n, k) in enumerate(shapes):
    g.manual_seed(1234 + 7919 * li)
    layers.append(lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128))


def acts(outliers):
    xs = {}
    for k in (8192, 28672):
        g.manual_seed(99 + k)
        x = torch.randn(M, k, generator=g, device="cuda")
        if outliers:
            mask = torch.rand(M, k, generator=g, device="cuda") < 1e-3
            x[mask] *= 20
        xs[k] = lqg.quantize_activations(x)
    return xs


ys = [torch.empty(M, n, dtype=torch.bfloat16, device="cuda") for n, _ in shapes]
ws = lqg.Workspace(0)


def graph(xs):
    def step():
        for (n, k), dw, y in zip(shapes, layers, ys):
            q, ts = xs[k]
            dw.gemm(q, ts, out=y, workspace=ws)
    step()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    gr.replay()
    torch.cuda.synchronize()
    return gr


def timed(gr, reps=5):
    samples, stop = [], [False]

    def sampler():
        while not stop[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(H) / 1000.0))
            time.sleep(0.005)
    t = threading.Thread(target=sampler)
    t.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    t.join()
    us = e0.elapsed_time(e1) / (reps * 3) * 1e3
    clk = sorted(s[0] for s in samples) or [0]
    pw = sorted(s[1] for s in samples) or [0]
    return us, clk[len(clk) // 2], pw[len(pw) // 2], pw[-1]


for name, outl in (("plain", False), ("outliers", True)):
    gr = graph(acts(outl))
    time.sleep(2.0)
    us, c, p, pmax = timed(gr)
    print(f"{name:9s} after idle : {us:8.1f} us  sm {c} MHz  power median {p:.0f} W max {pmax:.0f} W")
    t0 = time.time()
    while time.time() - t0 < 8:
        gr.replay()
    torch.cuda.synchronize()
    us, c, p, pmax = timed(gr)
    print(f"{name:9s} after heat : {us:8.1f} us  sm {c} MHz  power median {p:.0f} W max {pmax:.0f} W")
print("power limit", pynvml.nvmlDeviceGetEnforcedPowerLimit(H) / 1000.0, "W")

"""Why does the bench sweep's decode differ from tools/ab.py? Time the M=16
4-layer graph under progressively bench-like conditions."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_01229_b200 as lqg
shapes = [(10240, 8192), (8192, 8192), (28672, 8192), (8192, 28672)]
g = torch.Generator(device="cuda"); g.manual_seed(1)
layers = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128) for n, k in shapes]
ws = lqg.Workspace(0)

def timeit(m, xs, ys, tag):
    def step():
        for (n, k), dw, y in zip(shapes, layers, ys):
            q, ts = xs[k]
            dw.gemm(q[:m], ts[:m], out=y[:m], workspace=ws)
    step(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        for _ in range(3): step()
    torch.cuda.current_stream().wait_stream(s)
    gr.replay(); torch.cuda.synchronize()
    out = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3): gr.replay()
        e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / 9 * 1e3)
    print(f"{tag:40s} M={m}: {statistics.median(out):.1f} us")

for rows in (16, 4096):
    xs = {k: lqg.quantize_activations(torch.randn(rows, k, generator=g, device="cuda")) for k in (8192, 28672)}
    ys = [torch.empty(rows, n, dtype=torch.bfloat16, device="cuda") for n, _ in shapes]
    for m in (1, 16):
        timeit(m, xs, ys, f"x rows={rows}")
# now run big-M launches first (like the bench's full step), then decode again
for m in (4096, 1024):
    timeit(m, xs, ys, "big M")
import time
for m in (1, 16):
    timeit(m, xs, ys, "after big M")
for pause in (1, 3, 10):
    time.sleep(pause)
    timeit(16, xs, ys, f"after big M + {pause}s idle")
try:
    import pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("sm", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), "mem", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
          "temp", pynvml.nvmlDeviceGetTemperature(h, 0), "reasons", hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
except Exception as e:
    print("nvml", e)

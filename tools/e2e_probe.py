"""The e2e step (bench.py's `e2e`: 52 synchronous host-buffer calls
lqg_gemm_w4a8_host over the 70B sweep) under host-call chunking knobs, next
to the raw pinned PCIe bandwidth of this box.

  python tools/e2e_probe.py ["host_chunk_m=2048,host_chunks=8" ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg
from bench import WORKLOADS, algo_ops

dev = torch.device("cuda", 0)
# raw PCIe: pinned 512 MB each way, alone and concurrently
a = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
b = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
c = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
for name, fn in (("H2D", lambda: b.copy_(a, non_blocking=True)), ("D2H", lambda: c.copy_(b, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"pinned {name}: {a.numel() / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
b2 = torch.empty_like(b)
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    b2.copy_(a, non_blocking=True)
with torch.cuda.stream(s2):
    c.copy_(b, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"pinned H2D + D2H concurrently: {2 * a.numel() / dt / 1e9:.1f} GB/s total")
del a, b, c, b2

wl = WORKLOADS["llama2-70b"]
ms = wl["m_sweep"]
g = torch.Generator(device=dev).manual_seed(0)
layers = []
for name, n, k in wl["shapes"]:
    layers.append((name, n, k, lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device=dev) * 0.02, 128)))
hx = {}
for k in {k for _, _, k in wl["shapes"]}:
    q, ts = lqg.quantize_activations(torch.randn(max(ms), k, generator=g, device=dev))
    hx[k] = (q.cpu().pin_memory(), ts.cpu().pin_memory())
hy = {name: torch.empty(max(ms), n, dtype=torch.bfloat16).pin_memory() for name, n, _, _ in layers}
ops = sum(algo_ops(m, n, k) for m in ms for _, n, k, _ in layers)


def step():
    for m in ms:
        for name, n, k, dw in layers:
            qh, th = hx[k]
            dw.gemm_host(qh[:m], th[:m], hy[name][:m])


for cfg in (sys.argv[1:] or [""]):
    knobs = dict(kv.split("=") for kv in cfg.split(",") if kv)
    with lqg.tune(**{kk: int(v) for kk, v in knobs.items()}):
        step()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            step()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
    print(f"e2e [{cfg or 'default'}]: {best * 1e3:.2f} ms/step = {ops / best / 1e12:.1f} TOPS")

# per-M breakdown of the default configuration: time of the 4 calls, their
# PCIe bytes, and the effective transfer rate
print("   M    ms   H2D MB   D2H MB   GB/s (H2D+D2H over the calls' time)")
for m in ms:
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for name, n, k, dw in layers:
            qh, th = hx[k]
            dw.gemm_host(qh[:m], th[:m], hy[name][:m])
        best = min(best, time.perf_counter() - t0)
    h2d = sum(m * k + 4 * m for _, n, k, _ in layers)
    d2h = sum(2 * m * n for _, n, k, _ in layers)
    print(f"{m:5d} {best * 1e3:6.3f} {h2d / 1e6:8.1f} {d2h / 1e6:8.1f} {(h2d + d2h) / best / 1e9:7.1f}")

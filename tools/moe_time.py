"""Mixtral-8x7B expert FFN GEMMs (BASELINE config 5): one grouped launch vs one
launch per expert, device time of CUDA-graph replays (weights 8 x 29 MB per
layer exceed L2 between replays).
  python tools/moe_time.py [tokens ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_01229_b200 as lqg

E = 8
shapes = {"w1": (14336, 4096), "w2": (4096, 14336)}
toks = [int(t) for t in sys.argv[1:]] or [1, 8, 64, 512, 4096]
g = torch.Generator(device="cuda").manual_seed(0)
experts = {nm: [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
                for _ in range(E)] for nm, (n, k) in shapes.items()}
ws = lqg.Workspace(0)


def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        for _ in range(reps):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


rng = np.random.default_rng(0)
for T in toks:
    # top-2 routing of T tokens over 8 experts (skewed like a real router)
    p = rng.dirichlet(np.full(E, 2.0))
    ms = np.bincount(rng.choice(E, size=2 * T, p=p), minlength=E).astype(np.uint32).tolist()
    rows = sum(ms)
    for nm, (n, k) in shapes.items():
        dws = experts[nm]
        xq, ts = lqg.quantize_activations(torch.randn(rows, k, generator=g, device="cuda"))
        y = torch.empty(rows, n, dtype=torch.bfloat16, device="cuda")
        tg = timeit(lambda: lqg.gemm_grouped(dws, xq, ts, ms, out=y, workspace=ws))
        def per():
            r0 = 0
            for dw, m in zip(dws, ms):
                if m:
                    dw.gemm(xq[r0:r0 + m], ts[r0:r0 + m], out=y[r0:r0 + m], workspace=ws)
                r0 += m
        tp = timeit(per)
        wbytes = sum(dw.device_bytes for dw, m in zip(dws, ms) if m)
        ops = 2 * rows * n * k
        print(f"T={T:5d} {nm} rows={rows:5d} ms={ms}: grouped {tg:8.1f} us ({wbytes/tg/1e3:6.0f} GB/s, "
              f"{ops/tg/1e6:7.1f} TOPS) | per-expert {tp:8.1f} us  x{tp/tg:.2f}")

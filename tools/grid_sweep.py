import sys, os
sys.path.insert(0, '/root/repo')
import torch, time
import paper_2509_01229_b200 as lqg
shapes = [("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 28672, 8192), ("down", 8192, 28672)]
def tgraph(fn, R=12):
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(R): fn()
    torch.cuda.current_stream().wait_stream(s); g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / R * 1e3)
    return best
for name, n, k in shapes:
    dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128) for _ in range(3)]
    for m in (64, 128, 256):
        q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
        y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        it = [0]
        def fn():
            dws[it[0] % 3].gemm(q, ts, out=y); it[0] += 1
        res = {}
        for grid in (0, 64, 80, 96, 112, 128):
            lqg.tune_set("grid", grid)
            try:
                res[grid] = tgraph(fn)
            except Exception as e:
                res[grid] = float('nan')
        lqg.tune_set("grid", 0)
        print(f"{name:8s} m={m:4d} " + " ".join(f"g{g}={t:6.1f}" for g, t in res.items()), flush=True)

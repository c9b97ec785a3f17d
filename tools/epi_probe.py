"""Time one shape with INT32 / F32 / BF16 outputs (epilogue-cost probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_01229_b200 as lqg
n, k, m = map(int, sys.argv[1:4])
g = torch.Generator(device="cuda").manual_seed(0)
dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128) for _ in range(2)]
q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
outs = {"acc": torch.empty(m, n, dtype=torch.int32, device="cuda"),
        "f32": torch.empty(m, n, dtype=torch.float32, device="cuda"),
        "bf16": torch.empty(m, n, dtype=torch.bfloat16, device="cuda")}
for name, y in outs.items():
    def run():
        for dw in dws:
            if name == "acc":
                dw.gemm_accum(q, out=y)
            else:
                dw.gemm(q, ts, out=y)
    run(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        for _ in range(5): run()
    torch.cuda.current_stream().wait_stream(s); gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    print(f"{n}x{k} m={m} {name}: {t*1e6:.1f} us  {2*m*n*k/t/1e12:.0f} TOPS")

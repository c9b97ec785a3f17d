import sys, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2509_01229_b200 as lqg
fails = 0
for it in range(60):
    for m in (2048, 3001):
        g = torch.Generator(device="cuda").manual_seed(m + it)
        n, k = 384, 640
        dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        y_dev = dw.gemm(q, ts).cpu()
        y2 = dw.gemm(q, ts).cpu()
        qh, th = q.cpu().pin_memory(), ts.cpu().pin_memory()
        yh = torch.empty(m, n, dtype=torch.bfloat16).pin_memory()
        dw.gemm_host(qh, th, yh)
        if not torch.equal(yh, y_dev) or not torch.equal(y2, y_dev):
            fails += 1
            d = (yh != y_dev).nonzero()
            print("MISMATCH it", it, "m", m, "host-vs-dev", int((yh != y_dev).sum()), "dev-vs-dev", int((y2 != y_dev).sum()), d[:5].tolist())
print("fails", fails)

"""Repeat the CTA-pair vs one-CTA comparison (the large-token-tile split-K
paths) many times; report any mismatch. PS_QUAD=1: shapes that run in quad
mode (4-CTA clusters, DSMEM split-K exchange) -- pair (quad), pair with
no_quad=1 (L2 exchange) and one-CTA compared."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg

R = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
for it in range(R):
    cfgs = [(4096, 1024, 8192), (1000, 2048, 4096), (2048, 384, 640), (3001, 384, 640)]
    if os.environ.get("PS_ONLY"):
        cfgs = cfgs[:1]
    if os.environ.get("PS_QUAD"):
        cfgs = [(128, 8192, 2048), (64, 8192, 4096), (256, 4096, 4096), (128, 4096, 28672), (96, 2048, 1024)]
    for (m, n, k) in cfgs:
        g = torch.Generator(device="cuda").manual_seed(m + n + it)
        dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        outs = []
        extra = dict(kv.split("=") for kv in os.environ.get("PS_TUNE", "").split(",") if kv)
        variants = [dict(pair=0), dict(pair=1), dict(pair=-1)]
        if os.environ.get("PS_QUAD"):
            variants.append(dict(pair=1, no_quad=1))
        for var in variants:
            with lqg.tune(**var, **{kk: int(v) for kk, v in extra.items()}):
                outs.append((dw.gemm_accum(q), dw.gemm(q, ts)))
            if os.environ.get("PS_SYNC"):
                try:
                    torch.cuda.synchronize()
                except Exception as exc:
                    print(f"FAILED it={it} m={m} n={n} k={k} {var}: {exc}", flush=True)
                    raise
        torch.cuda.synchronize()
        for a, b in outs[1:]:
            if not (torch.equal(outs[0][0], a) and torch.equal(outs[0][1], b)):
                bad += 1
                d = (outs[0][0] != a).nonzero()
                print(f"MISMATCH it={it} m={m} n={n} k={k}: acc diffs {int((outs[0][0] != a).sum())} "
                      f"first {d[:4].tolist()}", flush=True)
print(f"pair_stress: {R} rounds, {bad} mismatches")

"""Repeat the CTA-pair vs one-CTA comparison and the pipelined host call (the
large-token-tile split-K paths) many times; report any mismatch."""
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
    for (m, n, k) in cfgs:
        g = torch.Generator(device="cuda").manual_seed(m + n + it)
        dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        outs = []
        extra = dict(kv.split("=") for kv in os.environ.get("PS_TUNE", "").split(",") if kv)
        for pair in (0, 1, -1):
            with lqg.tune(pair=pair, **{kk: int(v) for kk, v in extra.items()}):
                outs.append((dw.gemm_accum(q), dw.gemm(q, ts)))
            if os.environ.get("PS_SYNC"):
                try:
                    torch.cuda.synchronize()
                except Exception as exc:
                    print(f"FAILED it={it} m={m} n={n} k={k} pair={pair}: {exc}", flush=True)
                    raise
        torch.cuda.synchronize()
        for a, b in outs[1:]:
            if not (torch.equal(outs[0][0], a) and torch.equal(outs[0][1], b)):
                bad += 1
                d = (outs[0][0] != a).nonzero()
                print(f"MISMATCH it={it} m={m} n={n} k={k}: acc diffs {int((outs[0][0] != a).sum())} "
                      f"first {d[:4].tolist()}", flush=True)
print(f"pair_stress: {R} rounds, {bad} mismatches")

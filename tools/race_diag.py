"""Diagnose split-K mismatches: run the failing sequence, and on a mismatch in
the one-CTA kernel, express the wrong tile's error in terms of k-block range
partial sums (missing / doubled contributor pieces)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg

cfgs = [(4096, 1024, 8192), (1000, 2048, 4096), (2048, 384, 640), (3001, 384, 640)]
dws = {}
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    for ci, (m, n, k) in enumerate(cfgs):
        g = torch.Generator(device="cuda").manual_seed(m + n + it)
        dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        accs = {}
        for pair in (0, 1):
            with lqg.tune(pair=pair):
                accs[pair] = dw.gemm_accum(q)
            torch.cuda.synchronize()
        if torch.equal(accs[0], accs[1]):
            continue
        # reference: exact int mm of the dequantized weights
        wq = dw.dequant().to(torch.float64)        # [n, k]; float64 products are exact here
        ref = (q.to(torch.float64) @ wq.T).to(torch.int64).to(torch.int32)
        for pair in (0, 1):
            d = accs[pair] - ref
            bad = (d != 0).nonzero()
            if len(bad) == 0:
                print(f"it={it} cfg={ci} pair={pair}: correct")
                continue
            r0, c0 = bad.min(0).values.tolist()
            r1, c1 = bad.max(0).values.tolist()
            print(f"it={it} cfg={ci} pair={pair}: {len(bad)} wrong in rows [{r0},{r1}] cols [{c0},{c1}]")
            # explain the error over the bad block by k-block range partials
            blk = d[r0:r1 + 1, c0:c1 + 1]
            KB = (k + 255) // 256
            best = None
            for a in range(KB):
                for b in range(a + 1, KB + 1):
                    part = (q[r0:r1 + 1, a * 256:b * 256].to(torch.float64) @ wq[c0:c1 + 1, a * 256:b * 256].T).to(torch.int64).to(torch.int32)
                    for sgn in (1, -1):
                        if torch.equal(blk, sgn * part):
                            best = (sgn, a, b)
                            break
                    if best:
                        break
                if best:
                    break
            print("   error ==", f"{'+' if best[0] > 0 else '-'}partial(k-blocks {best[1]}..{best[2] - 1})" if best else "no single k-range partial")
print("done")

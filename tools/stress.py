"""GPU stress check: lqg accumulators vs torch._int_mm on the dequantized
weights, over many (n, k, m) configs and repeats. Debug tool (not a test)."""
import argparse
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_01229_b200 as lqg


def check(n, k, m, g=128, reps=3, seed=0):
    torch.manual_seed(seed)
    w = torch.randn(n, k, device="cuda") * 0.02
    dw = lqg.DeviceWeights.quantize(w, g)
    w8 = dw.dequant()
    x = torch.randn(m, k, device="cuda")
    q, ts = lqg.quantize_activations(x)
    mp = max(m, 32)
    qp = torch.zeros(mp, k, dtype=torch.int8, device="cuda")
    qp[:m] = q
    ref = torch._int_mm(qp, w8.t())[:m]
    bad = 0
    for r in range(reps):
        acc = dw.gemm_accum(q)
        torch.cuda.synchronize()
        d = (acc != ref).sum().item()
        bad += d
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="8192x28672x2048")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for c in a.configs.split(","):
        n, k, m = map(int, c.split("x"))
        try:
            bad = check(n, k, m, reps=a.reps)
            print(f"{c}: mismatches={bad}", flush=True)
        except Exception as e:
            print(f"{c}: ERROR {type(e).__name__}: {str(e).splitlines()[0]}", flush=True)
            return



def locate(n, k, m, g=128, seed=0, sms=148):
    """Print which (mt, nt) tiles mismatch and how stream-K split them."""
    torch.manual_seed(seed)
    w = torch.randn(n, k, device="cuda") * 0.02
    dw = lqg.DeviceWeights.quantize(w, g)
    w8 = dw.dequant()
    x = torch.randn(m, k, device="cuda")
    q, ts = lqg.quantize_activations(x)
    qp = torch.zeros(max(m, 32), k, dtype=torch.int8, device="cuda")
    qp[:m] = q
    ref = torch._int_mm(qp, w8.t())[:m]
    acc = dw.gemm_accum(q)
    torch.cuda.synchronize()
    MT = (m + 191) // 192
    BN = max(16, ((m + MT - 1) // MT + 15) // 16 * 16)
    NT = (n + 127) // 128
    KB = (k + 255) // 256
    total = MT * NT * KB
    G = min(sms, total)
    beg = [total * c // G for c in range(G + 1)]
    bad = (acc != ref).cpu()
    for mt in range(MT):
        for nt in range(NT):
            blk = bad[mt * BN:(mt + 1) * BN, nt * 128:(nt + 1) * 128]
            if blk.any():
                t = mt * NT + nt
                owners = [c for c in range(G) if beg[c] < (t + 1) * KB and beg[c + 1] > t * KB]
                rows = blk.any(dim=1).nonzero().flatten().tolist()
                print(f"tile mt={mt} nt={nt} t={t}: {int(blk.sum())} bad, owners={owners}, "
                      f"ranges={[(beg[c]-t*KB, beg[c+1]-t*KB) for c in owners]}, bad token rows {rows[:3]}..{rows[-3:]}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "locate":
        locate(*map(int, sys.argv[2].split("x")))
    else:
        main()

"""Small launches of every kernel variant, for compute-sanitizer runs
(memcheck / synccheck / racecheck / initcheck), each checked bit-exact against
the CPU oracle so a sanitizer-perturbed schedule is also a correctness run:

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Cases: decode (1 token tile, sentinel split-K), mid-M one-CTA kernel with the
flag + TMA-gather split-K, the CTA-pair kernel (cta_group::2, remote
mbarrier arrivals), the quad mode (4-CTA clusters, DSMEM split-K exchange),
a grouped (MoE) launch with an empty expert, the fan-out epilogue into two
destinations, and the GPU quantizers.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
import paper_2509_01229_b200 as lqg

port = oracle.Port()
rng = np.random.default_rng(5)
G = 128


def case(n, k, m, tune=None):
    w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    x = rng.standard_normal((m, k)).astype(np.float32)
    b = port.build_bundle_plain(w, G)
    q, ts = port.quantize_activations(x)
    acc_ref, y_ref = port.gemm_oracle(q, ts, port.bundle_int8(b), b["channel_scales"])
    bundle = lqg.QuantizedWeightBundle(n, k, G, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                       b["packed"], b["scales"], b["offsets"], b["channel_scales"])
    dw = lqg.DeviceWeights.from_bundle(bundle, 0)
    xq, tsd = torch.from_numpy(q).cuda(), torch.from_numpy(ts).cuda()
    with lqg.tune(**(tune or {})):
        acc = dw.gemm_accum(xq)
        y = dw.gemm(xq, tsd, out_dtype=torch.float32)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(acc.cpu().numpy().astype(np.int64), acc_ref)
    np.testing.assert_array_equal(y.cpu().numpy().view(np.uint32), y_ref.view(np.uint32))
    print(f"ok gemm n={n} k={k} m={m} {tune or ''}", flush=True)
    return dw, xq, tsd, y_ref


# decode: one 16-token tile, stream-K with sentinel split-K cells
case(1024, 4096, 16)
# mid-M, one-CTA kernel, 3 token chunks -> flag + TMA-gather split-K
case(1024, 4096, 48, tune=dict(pair=0))
# small weights at 96 tokens (auto_tile rule D): three 32-token tiles on the
# one-CTA kernel, sentinel split-K per tile
case(1024, 4096, 96)
# CTA pairs, two token tiles, ragged m
dw, xq, tsd, y_ref = case(1024, 2048, 200, tune=dict(pair=1, max_bn=128))
# quad mode: two CTA pairs per split tile in one 4-CTA cluster, DSMEM exchange
case(2048, 2048, 128, tune=dict(pair=1))
# fan-out epilogue: the same tile into two destinations
outs = [torch.empty(200, 1024, dtype=torch.float32, device="cuda") for _ in range(2)]
dw2, xq2, tsd2, y_ref2 = case(1024, 2048, 24)
dw2.gemm_fanout(xq2, tsd2, outs)
torch.cuda.synchronize()
for o in outs:
    np.testing.assert_array_equal(o[:24].cpu().numpy().view(np.uint32), y_ref2.view(np.uint32))
print("ok fanout", flush=True)
# grouped (MoE): 4 experts, one empty
ms = [5, 0, 40, 19]
n, k = 512, 2048
ws, refs, qs, tss = [], [], [], []
for e, me in enumerate(ms):
    w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    b = port.build_bundle_plain(w, G)
    ws.append(lqg.DeviceWeights.from_bundle(lqg.QuantizedWeightBundle(
        n, k, G, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(), b["packed"], b["scales"],
        b["offsets"], b["channel_scales"]), 0))
    x = rng.standard_normal((max(me, 1), k)).astype(np.float32)
    q, ts = port.quantize_activations(x)
    q, ts = q[:me], ts[:me]
    if me:
        refs.append(port.gemm_oracle(q, ts, port.bundle_int8(b), b["channel_scales"])[1])
    qs.append(q)
    tss.append(ts)
xq = torch.from_numpy(np.concatenate(qs)).cuda()
tsd = torch.from_numpy(np.concatenate(tss)).cuda()
y = lqg.gemm_grouped(ws, xq, tsd, ms, out_dtype=torch.float32)
torch.cuda.synchronize()
np.testing.assert_array_equal(y.cpu().numpy().view(np.uint32), np.concatenate(refs).view(np.uint32))
print("ok grouped", flush=True)
# GPU quantizers
w = (rng.standard_normal((256, 1024)) * 0.02).astype(np.float32)
dq = lqg.DeviceWeights.quantize(torch.from_numpy(w).cuda(), G).export()
np.testing.assert_array_equal(dq.packed_weights, port.build_bundle_plain(w, G)["packed"])
x = rng.standard_normal((7, 1024)).astype(np.float32)
q2, ts2 = lqg.quantize_activations(torch.from_numpy(x).cuda())
np.testing.assert_array_equal(q2.cpu().numpy(), port.quantize_activations(x)[0])
print("ok quantizers", flush=True)
print("ALL OK")

"""GPU parity of the grouped (MoE) W4A8 GEMM, lqg_gemm_w4a8_grouped: one
persistent launch over several experts that share n, k and group size (the
paper's MoE case; BASELINE config 5, Mixtral-8x7B expert FFNs).

Bar: per expert, INT32 accumulators bit-exact against the CPU oracle
(gemm.cpp:225-243) and F32 bit-identical to the reference epilogue
(quant.cpp:125-127); at Mixtral sizes, byte-identical to one lqg_gemm_w4a8
launch per expert (itself oracle-checked in test_gemm_gpu.py)."""
import numpy as np
import pytest

from conftest import make_acts, make_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "the gpu suite needs a B200"
    return torch


def _bundle(lqg, b):
    return lqg.QuantizedWeightBundle(b["n"], b["k"], b["group_size"], lqg.WeightLayout(b["layout"]),
                                     lqg.FragmentDescriptor(), b["packed"], b["scales"],
                                     b["offsets"], b["channel_scales"])


@pytest.mark.parametrize("ms,n,k,g", [
    ([3, 0, 17, 40], 256, 512, 128),
    ([1, 1, 1, 1, 1, 1, 1, 1], 384, 1024, 64),
    ([200, 5, 0, 193], 128, 768, 128),
    ([0, 0, 9], 100, 256, 32),
    ([450], 256, 256, 128),
])
def test_grouped_matches_oracle(torch_cuda, lqg, port, ms, n, k, g):
    torch = torch_cuda
    rng = np.random.default_rng(sum(ms) + n + k + g)
    bundles = [port.build_bundle_plain(make_weights(rng, n, k), g) for _ in ms]
    dws = [lqg.DeviceWeights.from_bundle(_bundle(lqg, b), 0) for b in bundles]
    rows = sum(ms)
    q, ts = port.quantize_activations(make_acts(rng, rows, k))
    xq = torch.from_numpy(q).cuda()
    tsd = torch.from_numpy(ts).cuda()
    acc = lqg.gemm_grouped_accum(dws, xq, ms).cpu().numpy()
    y = lqg.gemm_grouped(dws, xq, tsd, ms, out_dtype=torch.float32).cpu().numpy()
    yb = lqg.gemm_grouped(dws, xq, tsd, ms, out_dtype=torch.bfloat16).cpu()
    r0 = 0
    for b, m in zip(bundles, ms):
        if m:
            acc_ref, y_ref = port.gemm_oracle(q[r0:r0 + m], ts[r0:r0 + m], port.bundle_int8(b),
                                              b["channel_scales"])
            np.testing.assert_array_equal(acc[r0:r0 + m].astype(np.int64), acc_ref)
            np.testing.assert_array_equal(y[r0:r0 + m].view(np.uint32), y_ref.view(np.uint32))
            assert torch.equal(yb[r0:r0 + m], torch.from_numpy(y_ref).to(torch.bfloat16))
        r0 += m


@pytest.mark.parametrize("n,k,ms", [
    (14336, 4096, [9, 3, 0, 14, 6, 11, 1, 20]),          # Mixtral w1/w3, decode (64 tokens x top-2 / 2)
    (4096, 14336, [1, 2, 3, 4, 5, 6, 7, 8]),             # Mixtral w2, decode
    (4096, 14336, [600, 410, 512, 530, 470, 505, 540, 529]),  # w2, prefill (4096 tokens)
])
def test_grouped_mixtral_equals_per_expert_launches(torch_cuda, lqg, n, k, ms):
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(n + k + sum(ms))
    dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
           for _ in ms]
    rows = sum(ms)
    xq, ts = lqg.quantize_activations(torch.randn(rows, k, generator=g, device="cuda"))
    acc = lqg.gemm_grouped_accum(dws, xq, ms)
    y = lqg.gemm_grouped(dws, xq, ts, ms, out_dtype=torch.bfloat16)
    r0 = 0
    for dw, m in zip(dws, ms):
        if m:
            assert torch.equal(acc[r0:r0 + m], dw.gemm_accum(xq[r0:r0 + m]))
            assert torch.equal(y[r0:r0 + m], dw.gemm(xq[r0:r0 + m], ts[r0:r0 + m]))
        r0 += m
    # deterministic under stream-K (integer partials, any arrival order)
    assert torch.equal(acc, lqg.gemm_grouped_accum(dws, xq, ms))


def test_grouped_rejects_bad_groups(torch_cuda, lqg):
    torch = torch_cuda
    a = lqg.DeviceWeights.quantize(torch.randn(128, 256, device="cuda"), 128)
    b = lqg.DeviceWeights.quantize(torch.randn(256, 256, device="cuda"), 128)
    xq = torch.zeros(4, 256, dtype=torch.int8, device="cuda")
    ts = torch.ones(4, device="cuda")
    with pytest.raises(lqg.ValidationError, match="share n, k"):
        lqg.gemm_grouped([a, b], xq, ts, [2, 2])
    with pytest.raises(lqg.ValidationError, match="sum of group token counts"):
        lqg.gemm_grouped([a, a], xq, ts, [1, 2])
    with pytest.raises(lqg.ValidationError, match=">= 1"):
        lqg.gemm_grouped([a, a], xq[:0], ts[:0], [0, 0])


@pytest.mark.parametrize("ms,n,k", [([700, 0, 333, 1200, 5], 1024, 2048), ([321, 322], 512, 4096)])
def test_grouped_pair_mode_equals_one_cta(torch_cuda, lqg, ms, n, k):
    """Grouped launches use CTA pairs from 320 tokens in the largest group;
    bit-identical to the one-CTA grouped kernel (tune pair=0)."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(sum(ms) + n)
    dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128) for _ in ms]
    xq, ts = lqg.quantize_activations(torch.randn(sum(ms), k, generator=g, device="cuda"))
    res = {}
    for mode in ("0", "1"):
        with lqg.lq.tune(pair=int(mode)):
            res[mode] = (lqg.gemm_grouped_accum(dws, xq, ms), lqg.gemm_grouped(dws, xq, ts, ms))
            torch.cuda.synchronize()
    assert torch.equal(res["0"][0], res["1"][0]) and torch.equal(res["0"][1], res["1"][1])

"""GPU parity tests: the sm_100a kernels against the CPU oracle, through the
C ABI (include/lqg.h). Bar: bit-exact INT32 accumulators and INT8 weights,
F32 output bit-identical to the reference epilogue, F16/BF16 = RNE of it."""
import numpy as np
import pytest

from conftest import make_acts, make_weights

pytestmark = pytest.mark.gpu


def to_bundle(lqg, b: dict):
    return lqg.QuantizedWeightBundle(b["n"], b["k"], b["group_size"], lqg.WeightLayout(b["layout"]),
                                     lqg.FragmentDescriptor(), b["packed"], b["scales"],
                                     b["offsets"], b["channel_scales"])


SHAPES = [
    # m, n, k, g
    (1, 128, 128, 128),
    (16, 128, 256, 128),
    (16, 256, 4096, 128),
    (5, 64, 64, 64),
    (33, 192, 384, 64),
    (100, 320, 512, 32),
    (257, 128, 256, 128),
    (300, 384, 640, 128),
    (1, 4096, 4096, 128),
    (16, 4096, 4096, 128),
    (64, 1024, 2048, 256),
]


@pytest.mark.parametrize("m,n,k,g", SHAPES)
def test_accum_and_f32_bit_exact(lqg, port, m, n, k, g):
    import torch
    rng = np.random.default_rng(1000 + m + n + k + g)
    w = make_weights(rng, n, k)
    b = port.build_bundle_plain(w, g)
    x = make_acts(rng, m, k)
    q, ts = port.quantize_activations(x)
    w_i8 = port.bundle_int8(b)
    acc_ref, y_ref = port.gemm_oracle(q, ts, w_i8, b["channel_scales"])

    dw = lqg.DeviceWeights.from_bundle(to_bundle(lqg, b), 0)
    xq = torch.from_numpy(q).cuda()
    tsd = torch.from_numpy(ts).cuda()
    acc = dw.gemm_accum(xq).cpu().numpy()
    np.testing.assert_array_equal(acc.astype(np.int64), acc_ref)
    y = dw.gemm(xq, tsd, out_dtype=torch.float32).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), y_ref.view(np.uint32))
    for dt in (torch.float16, torch.bfloat16):
        yl = dw.gemm(xq, tsd, out_dtype=dt).cpu()
        expect = torch.from_numpy(y_ref).to(dt)
        assert torch.equal(yl, expect)
    # dequantized INT8 weights through the mainloop's LQQ routine
    np.testing.assert_array_equal(dw.dequant().cpu().numpy(), w_i8)

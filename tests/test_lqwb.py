"""LQWB bundle files (§8 f-2): the reference's on-disk format (bundle.hpp:5-24,
save_bundle / load_bundle, bundle.cpp:137-224) into device handles.

Fixtures in tests/golden/lqwb were written and judged by the UNMODIFIED
reference (oracle/gen_lqwb.py): lqg must accept exactly the files the
reference's load_bundle accepts and reject the others with the same status and
message. The GPU half checks that a loaded file holds the reference's logical
codes and parameters (device prepack) and computes bit-exact GEMMs, and that
lqg_weights_save writes a file the reference reads back identically."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import make_acts

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "lqwb")
EXPECTED = json.load(open(os.path.join(GOLD, "expected.json")))


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_file_verdicts_match_reference(lqg, name):
    """Host-only read_bundle checks (no GPU): same status code and message."""
    code, msg = EXPECTED[name]
    L = lqg._lib.lib()
    path = os.path.join(GOLD, name)
    rc = L.lqg_bundle_file_validate(os.fsencode(path))
    got = L.lqg_last_error().decode().replace(GOLD + os.sep, "")
    assert rc == code, (rc, got)
    if code:
        assert got == msg


@pytest.mark.parametrize("name", [n for n, (c, _) in sorted(EXPECTED.items()) if c == 3 and n != "missing.lqwb"])
def test_truncated_files_raise_ioerror_with_offset(lqg, name):
    """The Python mirror raises lq::IoError with the reference's message and
    byte offset (errors.hpp:23-28), the suffix appearing once."""
    _, msg = EXPECTED[name]
    with pytest.raises(lqg.IoError) as ei:
        lqg.DeviceWeights.load(os.path.join(GOLD, name))
    assert str(ei.value) == msg
    assert ei.value.byte_offset == int(msg.rsplit(" ", 1)[1].rstrip(")"))


def test_load_without_gpu_fails_loudly(lqg):
    """A valid file still needs an sm_100 device to become a handle."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = lqg._lib.lib()
    h = C.c_void_p()
    rc = L.lqg_weights_load(os.fsencode(os.path.join(GOLD, "plain.lqwb")), 0, C.byref(h))
    assert rc == 6  # LQG_EUNSUPPORTED


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["plain", "dual"])
def test_load_holds_reference_bundle_and_gemm_is_exact(lqg, port, name):
    import torch
    f = np.load(os.path.join(GOLD, f"{name}.npz"))
    n, k, g = int(f["n"]), int(f["k"]), int(f["g"])
    dw = lqg.DeviceWeights.load(os.path.join(GOLD, f"{name}.lqwb"), 0)
    assert (dw.n, dw.k, dw.group_size) == (n, k, g)
    e = dw.export()
    np.testing.assert_array_equal(port.logical_codes(n, k, 0, e.packed_weights), f["codes"].reshape(n, k))
    np.testing.assert_array_equal(e.group_scales, f["scales"])
    np.testing.assert_array_equal(e.group_offsets, f["offsets"])
    np.testing.assert_array_equal(e.channel_scales.view(np.uint32), f["channel_scales"].view(np.uint32))
    rng = np.random.default_rng(7)
    q, ts = port.quantize_activations(make_acts(rng, 37, k))
    w8 = port.reconstruct_int8(n, k, g, f["codes"].reshape(n, k), f["scales"].reshape(n, -1),
                               f["offsets"].reshape(n, -1))
    acc_ref, y_ref = port.gemm_oracle(q, ts, w8, f["channel_scales"])
    xq = torch.from_numpy(q).cuda()
    acc = dw.gemm_accum(xq).cpu().numpy()
    y = dw.gemm(xq, torch.from_numpy(ts).cuda(), out_dtype=torch.float32).cpu().numpy()
    np.testing.assert_array_equal(acc.astype(np.int64), acc_ref)
    np.testing.assert_array_equal(y.view(np.uint32), y_ref.view(np.uint32))


@pytest.mark.gpu
def test_device_prepack_equals_host_prepack(lqg, port):
    """Plain bundles are prepacked by prepack_plain_kernel; the image must be
    byte-identical to the host prepack (lqg_prepack_host) incl. padding."""
    import torch
    rng = np.random.default_rng(11)
    for n, k, g in [(200, 96 * 4, 32), (128, 512, 128), (77, 1024, 256)]:
        w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        b = port.build_bundle_plain(w, g)
        bundle = lqg.QuantizedWeightBundle(n, k, g, lqg.WeightLayout.PlainRowMajor,
                                           lqg.FragmentDescriptor(), b["packed"], b["scales"],
                                           b["offsets"], b["channel_scales"])
        host_img = bundle.prepack()
        dw = lqg.DeviceWeights.from_bundle(bundle, 0)
        # reload the host image as a second handle; identical GEMMs + dequant
        dw2 = lqg.DeviceWeights.from_image(host_img, b["channel_scales"], n, k, g, 0)
        assert torch.equal(dw.dequant(), dw2.dequant())
        q, ts = port.quantize_activations(make_acts(rng, 19, k))
        xq = torch.from_numpy(q).cuda()
        assert torch.equal(dw.gemm_accum(xq), dw2.gemm_accum(xq))


@pytest.mark.gpu
def test_save_roundtrip_and_reference_reads_it(lqg, tmp_path):
    import torch
    import oracle
    dw = lqg.DeviceWeights.quantize(torch.randn(192, 512, device="cuda") * 0.02, 64)
    path = str(tmp_path / "w.lqwb")
    dw.save(path)
    dw2 = lqg.DeviceWeights.load(path, 0)
    a, b = dw.export(), dw2.export()
    for x, y in ((a.packed_weights, b.packed_weights), (a.group_scales, b.group_scales),
                 (a.group_offsets, b.group_offsets), (a.channel_scales, b.channel_scales)):
        np.testing.assert_array_equal(x, y)
    if oracle.ref_available():
        rb = oracle.Ref().load_bundle(path)
        arr = rb.arrays()
        np.testing.assert_array_equal(arr["packed"], a.packed_weights)
        np.testing.assert_array_equal(arr["channel_scales"], a.channel_scales)

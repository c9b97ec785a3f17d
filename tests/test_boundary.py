"""CPU: the drop-in boundary. liblqg.so loads and exports every symbol
include/lqg.h declares; host-side validation mirrors the reference
(bundle.cpp:89-135, gemm.cpp:11-17); the host prepack emits the documented
device layout (lqg_layout.h) for both reference layouts; and the product has
no CPU fallback (compute entry points fail loudly without an sm_100 GPU)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lqg.h")).read()
    return sorted(set(re.findall(r"\b(lqg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lqg):
    L = lqg._lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"liblqg.so does not export {s}"
    assert sorted(lqg._lib.EXPORTS) == syms


def test_library_is_sm100a_only(lqg):
    """The cubin in liblqg.so targets sm_100a and uses tcgen05 / TMA (SASS check)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", lqg._lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lqg._lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCIMMA", "STTM", "LDTM", "UBLKCP", "UTMALDG"):
        assert mnemonic in sass, mnemonic


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2509_01229_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "liblqoracle" not in txt and "liblqref" not in txt, f


def _bundle(lqg, port, n=64, k=128, g=64, layout=0, seed=0):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    b = port.build_bundle_plain(w, g)
    packed = b["packed"]
    if layout == 1:
        packed = port.pack_dual(port.logical_codes(n, k, 0, b["packed"]))
    return lqg.QuantizedWeightBundle(n, k, g, lqg.WeightLayout(layout), lqg.FragmentDescriptor(),
                                     packed, b["scales"].copy(), b["offsets"].copy(),
                                     b["channel_scales"].copy())


@pytest.mark.parametrize("mutate,match", [
    (lambda b: b.group_scales.__setitem__(3, 0), r"group scale 0 out of \[1,16\] at row 1 group 1"),
    (lambda b: b.group_offsets.__setitem__(0, 248), r"group offset 248 out of \[9,247\] at row 0 group 0"),
    (lambda b: b.channel_scales.__setitem__(5, np.inf), "channel scale at row 5 must be positive and finite"),
    (lambda b: setattr(b, "packed_weights", b.packed_weights[:-1]), "packed weight payload has wrong size"),
    (lambda b: setattr(b, "group_size", 48), "k = 128 not divisible by group_size = 48"),
    (lambda b: setattr(b, "n", 0), "bundle dimensions must be >= 1"),
])
def test_bundle_validation_mirrors_reference(lqg, port, ref, mutate, match):
    b = _bundle(lqg, port)
    mutate(b)
    with pytest.raises(lqg.ValidationError, match=match):
        b.validate()
    # the reference raises the same ValidationError text (bundle.cpp:89-135)
    import oracle
    if b.n >= 1:
        rb = ref.bundle_from_arrays(dict(n=b.n, k=b.k, group_size=b.group_size, layout=int(b.layout),
                                         packed=b.packed_weights, scales=b.group_scales,
                                         offsets=b.group_offsets, channel_scales=b.channel_scales))
        with pytest.raises(oracle.OracleError, match=match) as ei:
            ref.validate(rb)
        assert ei.value.code == 1


def test_dual_layout_validation(lqg, port):
    b = _bundle(lqg, port, n=64, k=128, g=64, layout=1)
    b.validate()
    b.group_size = 32
    b.group_scales = np.ones(64 * 4, np.uint8)
    b.group_offsets = np.full(64 * 4, 128, np.uint8)
    with pytest.raises(lqg.ValidationError, match="dual-MMA layout needs group_size divisible by 64"):
        b.validate()


def test_tile_config_rules(lqg, port):
    """gemm.cpp:11-17 (TileConfig::validate) and the packed-engine k_t rule."""
    dual = _bundle(lqg, port, layout=1)
    lqg.TileConfig(64, 64, 64).validate(dual)
    with pytest.raises(lqg.ValidationError, match="multiple of 64"):
        lqg.TileConfig(64, 64, 32).validate(dual)
    with pytest.raises(lqg.ValidationError, match="tile extents must be >= 1"):
        lqg.TileConfig(0, 64, 64).validate(dual)


def decode_image(img, n, k, g):
    """Python restatement of the documented device layout (lqg_layout.h)."""
    KBLK, TN = 256, 128
    P = 1 if g % 256 == 0 else 2 if g % 128 == 0 else 4 if g % 64 == 0 else 8
    chunk = TN * KBLK // 2 + 256 * P
    NT, KB = -(-n // TN), -(-k // KBLK)
    assert img.size == NT * KB * chunk
    ch = img.reshape(NT, KB, chunk)
    codes_raw = ch[:, :, :TN * KBLK // 2].reshape(NT, KB, 8, TN, 4, 4)  # nt kb c r word byte
    lo = codes_raw & 0xF
    hi = codes_raw >> 4
    # element 8w+j in lo nibble of byte j, 8w+j+4 in hi nibble
    el = np.concatenate([lo, hi], axis=-1)                               # nt kb c r w 8
    el = el.transpose(0, 3, 1, 2, 4, 5).reshape(NT * TN, KB * KBLK)       # row, k
    prm = ch[:, :, TN * KBLK // 2:].reshape(NT, KB, TN, P, 2)              # nt kb r p {s, a}
    s = prm[..., 0].transpose(0, 2, 1, 3).reshape(NT * TN, KB * P)
    a = prm[..., 1].transpose(0, 2, 1, 3).reshape(NT * TN, KB * P)
    return el[:n, :k], s, a, P


@pytest.mark.parametrize("n,k,g,layout", [(64, 128, 64, 0), (64, 128, 64, 1), (200, 384, 128, 0),
                                          (128, 256, 256, 1), (3, 96, 32, 0), (130, 512, 128, 1)])
def test_host_prepack_layout(lqg, port, n, k, g, layout):
    """lqg_prepack_host on either reference layout encodes exactly the bundle's
    logical codes and group params (parity on logical codes, bundle.cpp:227-249),
    with padding that dequantizes to 0."""
    if layout == 1 and (n % 64 or k % 64 or g % 64):
        pytest.skip("dual layout needs n, k, g multiples of 64")
    b = _bundle(lqg, port, n, k, g, layout, seed=n + k)
    img = b.prepack()
    codes, s, a, P = decode_image(img, n, k, g)
    want = port.logical_codes(n, k, layout, b.packed_weights)
    np.testing.assert_array_equal(codes, want)
    gpr = k // g
    sub = 256 // P
    for kb_p in range(s.shape[1]):
        k0 = kb_p * sub
        if k0 >= k:
            assert (s[:, kb_p] == 1).all() and (a[:, kb_p] == 128).all()
            continue
        gi = k0 // g
        np.testing.assert_array_equal(s[:n, kb_p], b.group_scales.reshape(n, gpr)[:, gi])
        np.testing.assert_array_equal(a[:n, kb_p], b.group_offsets.reshape(n, gpr)[:, gi])
    assert (s[n:] == 1).all() and (a[n:] == 128).all()


def test_prepack_rejects_unsupported_group_size(lqg, port):
    b = _bundle(lqg, port, n=2, k=96, g=32)
    b.group_size = 48
    b.group_scales = np.ones(4, np.uint8)
    b.group_offsets = np.full(4, 128, np.uint8)
    b.validate()  # the reference accepts g = 48 ...
    with pytest.raises(lqg.ValidationError, match="group_size % 32 == 0"):
        b.prepack()  # ... the device layout does not


def test_no_cpu_fallback(lqg, port):
    """Without an sm_100 device every compute entry point raises; nothing
    silently computes on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu suite")
    b = _bundle(lqg, port)
    with pytest.raises(lqg.UnsupportedDeviceError):
        lqg.DeviceWeights.from_bundle(b, 0)
    act = lqg.ActivationQuant(1, 128, np.zeros(128, np.int8), np.ones(1, np.float32))
    with pytest.raises((lqg.UnsupportedDeviceError, RuntimeError, AssertionError)):
        lqg.gemm_w4a8(act, b)

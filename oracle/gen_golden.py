"""TEST INFRASTRUCTURE ONLY — generates tests/golden/*.npz from the UNMODIFIED
reference library (oracle/_ref/liblqref.so, built by oracle/Makefile from
/root/reference/proj/src). Run in the container that has /root/reference:

    python -m oracle.gen_golden

Every array in the fixtures is an output of the reference itself; inputs are
seeded numpy draws stored alongside. The fixtures pin both the C restatement
(tests/test_oracle.py) and the GPU kernels (tests/test_gemm_gpu.py).
"""
from __future__ import annotations

import os

import numpy as np

import oracle

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def quant_cases(ref: oracle.Ref) -> dict:
    """build_bundle (quant.cpp:203-232) on small matrices incl. edge rows."""
    rng = np.random.default_rng(20240901)
    out = {}
    cases = [(4, 128, 64), (3, 256, 128), (2, 96, 32), (64, 128, 64), (128, 256, 128)]
    for ci, (n, k, g) in enumerate(cases):
        w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        if ci == 0:
            w[0] = 0.0                      # all-zero row -> s = 1
            w[1] = 60.0                     # constant row -> codes 0, offset 247
            w[2, :64] = np.linspace(-1, 1, 64, dtype=np.float32)  # full-span group
        if ci == 1:
            w[0, :3] = [1e-30, -1e-30, 5.0]  # tiny values next to a large one
        rb = ref.build_bundle(w, g, 0)
        a = rb.arrays()
        out[f"q{ci}_w"] = w
        out[f"q{ci}_g"] = np.int32(g)
        for key in ("packed", "scales", "offsets", "channel_scales"):
            out[f"q{ci}_{key}"] = a[key]
        out[f"q{ci}_codes"] = ref.logical_codes(rb)
        out[f"q{ci}_w_i8"] = ref.reconstruct_int8(rb)
        if n % 64 == 0 and k % 64 == 0 and g % 64 == 0:
            out[f"q{ci}_dual_packed"] = ref.to_dual(rb).arrays()["packed"]
    out["n_cases"] = np.int32(len(cases))
    return out


def act_cases(ref: oracle.Ref) -> dict:
    """quantize_activations_per_token (gemm.cpp:19-47)."""
    rng = np.random.default_rng(7)
    out = {}
    xs = [np.array([[2.0, -4.0], [0.0, 0.0]], np.float32),           # test_gemm.cpp:176-186
          rng.standard_normal((8, 256)).astype(np.float32),
          (rng.standard_normal((5, 64)) * 1e-3).astype(np.float32)]
    x3 = rng.standard_normal((4, 128)).astype(np.float32)
    x3[1, 7] = 50.0                                                   # outlier token
    x3[2] = 0.0
    xs.append(x3)
    for i, x in enumerate(xs):
        q, ts = ref.quantize_activations(x)
        out[f"a{i}_x"], out[f"a{i}_q"], out[f"a{i}_ts"] = x, q, ts
    out["n_cases"] = np.int32(len(xs))
    return out


def gemm_cases(ref: oracle.Ref) -> dict:
    """gemm_w4a8_accum / gemm_w4a8 (gemm.cpp:138-223) on small instances,
    including the acceptance-criterion-6 generator shape family
    (acceptance.cpp:265-315: m in [1,64], n = 64*[1..8], k = 64*[1..16], g = 64)."""
    rng = np.random.default_rng(66)
    specs = [  # m, n, k, g, layout
        (16, 128, 512, 128, 1), (1, 64, 64, 64, 0), (5, 192, 256, 64, 1), (33, 64, 768, 64, 0),
        (64, 512, 128, 64, 1), (12, 64, 128, 64, 1), (3, 100, 96, 32, 0), (7, 128, 512, 256, 0),
        (40, 192, 384, 64, 1), (257, 64, 128, 64, 0),
    ]
    for _ in range(6):
        m = int(rng.integers(1, 65))
        n = 64 * int(rng.integers(1, 5))
        k = 64 * int(rng.integers(1, 9))
        specs.append((m, n, k, 64, int(rng.integers(0, 2))))
    out = {}
    for ci, (m, n, k, g, layout) in enumerate(specs):
        w = rng.uniform(-2, 2, (n, k)).astype(np.float32)
        x = rng.uniform(-2, 2, (m, k)).astype(np.float32)
        rb = ref.build_bundle(w, g, layout)
        a = rb.arrays()
        q, ts = ref.quantize_activations(x)
        tile = [(64, 64, 64), (32, 128, 128), (16, 256, 192)][ci % 3]
        if layout == 1 and tile[2] % 64:
            tile = (64, 64, 64)
        engine = 1 if (n % 64 == 0 and k % 64 == 0 and g % 64 == 0) else 0
        acc = ref.gemm_w4a8_accum(rb, q, ts, tile, engine=engine)
        y = ref.gemm_w4a8(rb, q, ts, tile, engine=engine)
        out[f"c{ci}_dims"] = np.array([m, n, k, g, layout], np.int32)
        for key in ("packed", "scales", "offsets", "channel_scales"):
            out[f"c{ci}_{key}"] = a[key]
        out[f"c{ci}_q"], out[f"c{ci}_ts"] = q, ts
        out[f"c{ci}_acc"], out[f"c{ci}_y"] = acc, y
        if ci < 3:
            out[f"c{ci}_w_i8"] = ref.reconstruct_int8(rb)
    out["n_cases"] = np.int32(len(specs))
    return out


def known_answer_gemms(ref: oracle.Ref) -> dict:
    """test_gemm.cpp:29-92 cases through the reference."""
    out = {}
    # constant 60.0 row x unit activation -> acc 127*119 (test_gemm.cpp:29-50)
    w = np.full((1, 64), 60.0, np.float32)
    rb = ref.build_bundle(w, 64, 0)
    x = np.zeros((1, 64), np.float32)
    x[0, 0] = 1.0
    q, ts = ref.quantize_activations(x)
    a = rb.arrays()
    out.update({f"const_{k}": v for k, v in a.items() if isinstance(v, np.ndarray)})
    out["const_q"], out["const_ts"] = q, ts
    out["const_acc"] = ref.gemm_w4a8_accum(rb, q, ts, (64, 64, 64), 0)
    out["const_y"] = ref.gemm_w4a8(rb, q, ts, (64, 64, 64), 0)
    # one-hot activations read back W^ (test_gemm.cpp:72-92)
    rng = np.random.default_rng(11)
    n, k = 64, 128
    w = rng.uniform(-3, 3, (n, k)).astype(np.float32)
    rb = ref.build_bundle(w, 64, 0)
    a = rb.arrays()
    out.update({f"onehot_{kk}": v for kk, v in a.items() if isinstance(v, np.ndarray)})
    q = np.eye(k, dtype=np.int8)
    ts = np.ones(k, np.float32)
    out["onehot_acc"] = ref.gemm_w4a8_accum(rb, q, ts, (64, 64, 64), 1)
    out["onehot_w_i8"] = ref.reconstruct_int8(rb)
    return out


def lane_cases(ref: oracle.Ref) -> dict:
    """The exhaustive 16 x 16 x 239 lane box (test_quant.cpp:101-117) and random
    interleaved words through the reference dequant_word (packed.cpp:63-71)."""
    box = np.zeros((16, 16, 239), np.uint8)
    for c in range(16):
        for s in range(1, 17):
            for a in range(9, 248):
                lo, _, _ = ref.dequant_word(c, s, a)
                box[c, s - 1, a - 9] = lo & 0xFF
    rng = np.random.default_rng(20240817)
    words = rng.integers(0, 2**32, 4096, dtype=np.uint64).astype(np.uint32)
    ss = rng.integers(1, 17, 4096).astype(np.uint8)
    aa = rng.integers(9, 248, 4096).astype(np.uint8)
    lo = np.zeros(4096, np.uint32)
    hi = np.zeros(4096, np.uint32)
    for i in range(4096):
        lo[i], hi[i], _ = ref.dequant_word(int(words[i]), int(ss[i]), int(aa[i]))
    return {"box_lo_lane0": box, "words": words, "s": ss, "a": aa, "lo": lo, "hi": hi}


def main():
    if not oracle.ref_available():
        oracle.build()
    ref = oracle.Ref()
    os.makedirs(OUT, exist_ok=True)
    for name, fn in [("quant", quant_cases), ("act", act_cases), ("gemm", gemm_cases),
                     ("known", known_answer_gemms), ("lanes", lane_cases)]:
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **fn(ref))
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()

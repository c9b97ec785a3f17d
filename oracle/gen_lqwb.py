"""TEST INFRASTRUCTURE ONLY — LQWB bundle-file fixtures from the UNMODIFIED
reference library (oracle/_ref/liblqref.so: lq::save_bundle / lq::load_bundle,
bundle.cpp:137-224). Run in the container that has /root/reference:

    python -m oracle.gen_lqwb

Writes tests/golden/lqwb/:
  * plain.lqwb, dual.lqwb      files written by the reference's save_bundle
                               (+ plain.npz / dual.npz: the reference's logical
                               codes, scales, offsets and channel scales);
  * bad_*.lqwb                 byte-edited variants (bad magic, version, layout
                               flag, zero dimension, truncations, trailing byte,
                               out-of-range group scale) and
  * expected.json              the reference load_bundle verdict for every file:
                               {"file": [status, message]} (0 ok, 1 validation,
                               3 I/O), which lqg_weights_load must reproduce.
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np

import oracle

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "lqwb")


def main() -> None:
    ref = oracle.Ref()
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20250904)
    files = {}
    for name, layout, (n, k, g) in (("plain", 0, (64, 256, 64)), ("dual", 1, (64, 256, 128))):
        w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        rb = ref.build_bundle(w, g, layout)
        path = os.path.join(OUT, f"{name}.lqwb")
        ref.save_bundle(rb, path)
        a = rb.arrays()
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), n=n, k=k, g=g, layout=layout,
                            codes=ref.logical_codes(rb), scales=a["scales"], offsets=a["offsets"],
                            channel_scales=a["channel_scales"], packed=a["packed"])
        files[name] = path

    base = open(files["plain"], "rb").read()
    hdr = 4 + 2 + 4 + 4 + 4 + 1  # magic, version, n, k, g, layout (plain: no descriptor)
    n, k, g = struct.unpack_from("<III", base, 6)
    packed_len, ng = n * k // 2, n * (k // g)
    variants = {
        "bad_magic": b"LQWX" + base[4:],
        "bad_version": base[:4] + struct.pack("<H", 2) + base[6:],
        "bad_layout": base[:18] + bytes([7]) + base[19:],
        "zero_n": base[:6] + struct.pack("<I", 0) + base[10:],
        "k_not_multiple": base[:10] + struct.pack("<I", k + 1) + base[14:],
        "trunc_header": base[:12],
        "trunc_packed": base[:hdr + packed_len // 2],
        "trunc_scales": base[:hdr + packed_len + 3],
        "trunc_channel": base[:len(base) - 6],
        "trailing": base + b"\x00",
        "bad_scale": base[:hdr + packed_len] + bytes([0]) + base[hdr + packed_len + 1:],
        "bad_offset": base[:hdr + packed_len + ng] + bytes([3]) + base[hdr + packed_len + ng + 1:],
        "bad_channel": base[:len(base) - 4] + struct.pack("<f", -1.0),
    }
    for name, data in variants.items():
        path = os.path.join(OUT, f"{name}.lqwb")
        with open(path, "wb") as f:
            f.write(data)
        files[name] = path
    expected = {}
    for name, path in sorted(files.items()):
        try:
            ref.load_bundle(path)
            expected[os.path.basename(path)] = [0, ""]
        except oracle.OracleError as e:
            expected[os.path.basename(path)] = [e.code, str(e)]
    # a file that does not exist
    try:
        ref.load_bundle(os.path.join(OUT, "missing.lqwb"))
    except oracle.OracleError as e:
        expected["missing.lqwb"] = [e.code, str(e).replace(OUT + os.sep, "")]
    with open(os.path.join(OUT, "expected.json"), "w") as f:
        json.dump(expected, f, indent=1, sort_keys=True)
    print(json.dumps(expected, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()

"""CPU: the C restatement of the reference (oracle/lq_oracle.c) pinned against
golden vectors produced by the unmodified reference (tests/golden/, made by
oracle/gen_golden.py) and against the reference's own known-answer tests
(/root/reference/proj/tests/*.cpp, cited per test)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


# ---------------------------------------------------------------- known answers
def test_interleave_known_answer(port):
    """test_packed.cpp:11-23: [1..8] -> 0x84736251 -> lo 0x04030201, hi 0x08070605."""
    w = port.pack_interleaved([1, 2, 3, 4, 5, 6, 7, 8])
    assert w == 0x84736251
    lo = w & 0x0F0F0F0F
    hi = (w >> 4) & 0x0F0F0F0F
    assert (lo, hi) == (0x04030201, 0x08070605)


def test_lane_madd_and_xor_known_answers(port):
    """test_packed.cpp:38-51 via dequant_word's arithmetic: lane_madd(0x01020304, 2, 0x10)
    = 0x12141618; lane_xor_msb(0xFF7F80F9) = 0x7FFF0079."""
    assert (0x01020304 * 2 + 0x10101010) & 0xFFFFFFFF == 0x12141618
    assert 0xFF7F80F9 ^ 0x80808080 == 0x7FFF0079
    # dequant_word = unpack + madd + xor, 7 instructions per 8 elements (packed.hpp:89-95)
    lo, hi, ninstr = port.dequant_word(0x84736251, 2, 0x10)
    assert ninstr == 7
    assert lo == ((0x04030201 * 2 + 0x10101010) ^ 0x80808080)
    assert hi == ((0x08070605 * 2 + 0x10101010) ^ 0x80808080)


def test_worked_lqq_example(port):
    """test_quant.cpp:88-99 / P:350-351: code 15, s 15, min -104 (a = 24) -> 121."""
    assert port.dequantize_scalar(15, 15, 24) == 121
    assert port.dequantize_lane(15, 15, 24) == 0x79


def test_extremal_group_params(port):
    """test_quant.cpp:57-86: span 238 -> s 16, a 9, codes 0/15; span 232 -> 15;
    233 -> 16; constant group -> s 1, codes 0."""
    g = np.zeros((1, 64), np.int8)
    g[0, 0], g[0, 1] = -119, 119
    codes, sc, of = port.quantize_second_level(g, 64)
    assert (sc[0], of[0], codes[0, 0], codes[0, 1]) == (16, 9, 0, 15)
    g = np.full((1, 64), -116, np.int8)
    g[0, 0] = 116
    assert port.quantize_second_level(g, 64)[1][0] == 15
    g = np.full((1, 64), -117, np.int8)
    g[0, 0] = 116
    assert port.quantize_second_level(g, 64)[1][0] == 16
    g = np.full((1, 64), 37, np.int8)
    codes, sc, of = port.quantize_second_level(g, 64)
    assert sc[0] == 1 and of[0] == 128 + 37 and not codes.any()
    assert port.dequantize_scalar(0, 1, 128 + 37) == 37


def test_lane_box_exhaustive(port):
    """test_quant.cpp:101-117 / acceptance crit 2: the XOR lane form equals the wide
    scalar form on all 16 x 16 x 239 points, and equals the reference's output."""
    box = load("lanes")["box_lo_lane0"]
    pts = 0
    for c in range(16):
        for s in range(1, 17):
            for a in range(9, 248):
                lane = port.dequantize_lane(c, s, a)
                assert lane == (port.dequantize_scalar(c, s, a) & 0xFF)
                assert lane == box[c, s - 1, a - 9]
                pts += 1
    assert pts == 16 * 16 * 239


def test_dequant_words_match_reference(port):
    """Random interleaved words through packed.cpp:63-71 (including carrying,
    unreachable parameter combinations: the 32-bit IMAD semantics must match)."""
    d = load("lanes")
    for w, s, a, lo, hi in zip(d["words"][:1024], d["s"][:1024], d["a"][:1024], d["lo"][:1024],
                               d["hi"][:1024]):
        got = port.dequant_word(int(w), int(s), int(a))
        assert got[:2] == (int(lo), int(hi))


def test_round_half_away(port):
    """quant.hpp:33-35."""
    for v, want in [(0.5, 1), (-0.5, -1), (1.4999, 1), (2.5, 3), (-2.5, -3), (0.0, 0)]:
        assert port.round_half_away(v) == want


# ---------------------------------------------------------------- golden vectors
def test_quantizer_matches_reference_golden(port):
    """build_bundle (quant.cpp:203-232): packed payload, group params, channel scales,
    logical codes, INT8 reconstruction and the dual-MMA payload, bit for bit."""
    d = load("quant")
    for ci in range(int(d["n_cases"])):
        w, g = d[f"q{ci}_w"], int(d[f"q{ci}_g"])
        b = port.build_bundle_plain(w, g)
        for key in ("packed", "scales", "offsets"):
            np.testing.assert_array_equal(b[key], d[f"q{ci}_{key}"], err_msg=f"case {ci} {key}")
        np.testing.assert_array_equal(b["channel_scales"].view(np.uint32),
                                      d[f"q{ci}_channel_scales"].view(np.uint32))
        n, k = w.shape
        codes = port.logical_codes(n, k, 0, b["packed"])
        np.testing.assert_array_equal(codes, d[f"q{ci}_codes"])
        np.testing.assert_array_equal(port.bundle_int8(b), d[f"q{ci}_w_i8"])
        if f"q{ci}_dual_packed" in d:
            np.testing.assert_array_equal(port.pack_dual(codes), d[f"q{ci}_dual_packed"])
            np.testing.assert_array_equal(port.logical_codes(n, k, 1, d[f"q{ci}_dual_packed"]), codes)


def test_reconstruction_error_bound(port):
    """acceptance crit 4: |reconstructed - level-1 code| <= 8."""
    rng = np.random.default_rng(411)
    for g in (64, 128):
        w = rng.normal(0, 0.1, (4, 256)).astype(np.float32)
        q, _ = port.quantize_first_level(w)
        codes, sc, of = port.quantize_second_level(q, g)
        rec = port.reconstruct_int8(4, 256, g, codes, sc, of)
        assert np.abs(rec.astype(int) - q.astype(int)).max() <= 8
        assert q.min() >= -119 and q.max() <= 119


def test_activation_quant_matches_reference_golden(port):
    """quantize_activations_per_token (gemm.cpp:19-47) incl. test_gemm.cpp:176-186
    ([2,-4] -> scale 4/127, codes 64/-127; zero row -> scale 1)."""
    d = load("act")
    for i in range(int(d["n_cases"])):
        q, ts = port.quantize_activations(d[f"a{i}_x"])
        np.testing.assert_array_equal(q, d[f"a{i}_q"])
        np.testing.assert_array_equal(ts.view(np.uint32), d[f"a{i}_ts"].view(np.uint32))
    q, ts = port.quantize_activations(np.array([[2.0, -4.0], [0.0, 0.0]], np.float32))
    assert q[0].tolist() == [64, -127] and ts[1] == 1.0


def test_gemm_oracle_matches_reference_golden(port):
    """gemm_w4a8_accum / gemm_w4a8 (gemm.cpp:138-223) on the acceptance-crit-6 family:
    the int64 oracle equals the reference's INT32 accumulators and float output."""
    d = load("gemm")
    for ci in range(int(d["n_cases"])):
        m, n, k, g, layout = d[f"c{ci}_dims"].tolist()
        b = dict(n=n, k=k, group_size=g, layout=layout, packed=d[f"c{ci}_packed"],
                 scales=d[f"c{ci}_scales"], offsets=d[f"c{ci}_offsets"],
                 channel_scales=d[f"c{ci}_channel_scales"])
        port.validate_bundle(b)
        w_i8 = port.bundle_int8(b)
        if f"c{ci}_w_i8" in d:
            np.testing.assert_array_equal(w_i8, d[f"c{ci}_w_i8"])
        acc, y = port.gemm_oracle(d[f"c{ci}_q"], d[f"c{ci}_ts"], w_i8, b["channel_scales"])
        np.testing.assert_array_equal(acc, d[f"c{ci}_acc"].astype(np.int64), err_msg=f"case {ci}")
        np.testing.assert_array_equal(y.view(np.uint32), d[f"c{ci}_y"].view(np.uint32))


def test_known_answer_gemms(port):
    """test_gemm.cpp:29-50 (constant row: acc = 127*119, y ~= 60) and 72-92
    (one-hot activations read back W^)."""
    d = load("known")
    b = dict(n=1, k=64, group_size=64, layout=0, packed=d["const_packed"],
             scales=d["const_scales"], offsets=d["const_offsets"],
             channel_scales=d["const_channel_scales"])
    acc, y = port.gemm_oracle(d["const_q"], d["const_ts"], port.bundle_int8(b), b["channel_scales"])
    assert acc[0, 0] == 127 * 119 == d["const_acc"][0, 0]
    assert abs(y[0, 0] - 60.0) < 60.0 * 1e-5
    np.testing.assert_array_equal(d["onehot_acc"], d["onehot_w_i8"].T.astype(np.int32))


def test_accumulator_range_guard(port):
    """gemm.cpp:53-57 / test_gemm.cpp:198-226: k = 133120 ok, 133184 rejected."""
    assert port.accumulator_range_ok(133120)
    assert not port.accumulator_range_ok(133184)


def test_validation_messages(port):
    """bundle.cpp:89-135 rules."""
    from oracle import OracleError
    b = dict(n=1, k=64, group_size=64, layout=0, packed=np.zeros(32, np.uint8),
             scales=np.array([17], np.uint8), offsets=np.array([128], np.uint8),
             channel_scales=np.ones(1, np.float32))
    with pytest.raises(OracleError, match=r"group scale 17 out of \[1,16\] at row 0 group 0"):
        port.validate_bundle(b)
    b["scales"][0], b["offsets"][0] = 1, 8
    with pytest.raises(OracleError, match=r"group offset 8 out of \[9,247\]"):
        port.validate_bundle(b)
    b["offsets"][0], b["channel_scales"][0] = 9, 0.0
    with pytest.raises(OracleError, match="channel scale at row 0 must be positive and finite"):
        port.validate_bundle(b)


# ---------------------------------------------------------------- live reference
@pytest.mark.parametrize("n,k,g", [(64, 128, 64), (128, 384, 128), (5, 96, 32), (192, 256, 64)])
def test_port_equals_live_reference(port, ref, n, k, g):
    """When oracle/_ref is built: the restatement equals the reference on fresh
    seeded inputs (quantizer, layouts, activation quant, GEMM)."""
    rng = np.random.default_rng(n * 1000 + k + g)
    w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    b = port.build_bundle_plain(w, g)
    rb = ref.build_bundle(w, g, 0)
    ra = rb.arrays()
    for key in ("packed", "scales", "offsets", "channel_scales"):
        np.testing.assert_array_equal(b[key], ra[key])
    x = rng.standard_normal((9, k)).astype(np.float32)
    q, ts = port.quantize_activations(x)
    q2, ts2 = ref.quantize_activations(x)
    np.testing.assert_array_equal(q, q2)
    acc, y = port.gemm_oracle(q, ts, port.bundle_int8(b), b["channel_scales"])
    np.testing.assert_array_equal(acc, ref.gemm_w4a8_accum(rb, q, ts, engine=0).astype(np.int64))
    np.testing.assert_array_equal(y, ref.gemm_w4a8(rb, q, ts, engine=0))
    if n % 64 == 0 and k % 64 == 0 and g % 64 == 0:
        codes = port.logical_codes(n, k, 0, b["packed"])
        np.testing.assert_array_equal(port.pack_dual(codes), ref.to_dual(rb).arrays()["packed"])


def test_b200_profile_through_reference_cost_model(ref):
    """profiles/b200.profile parses with the reference's parse_profile and puts
    the W4A8 regime flip where the measured sweep has it (M* ~ 120,
    cost_model.cpp:150-157); LiquidQuant's 7/8 op per element stays below the
    memory-bound alpha threshold."""
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "b200.profile")
    m_star, a_mem, a_comp = ref.profile_diag(path)
    assert 110 <= m_star <= 130
    assert a_mem > 7 / 8 and a_comp > 7 / 8
    t16, cb16 = ref.cost_total(path, 8192, 28672, 16, (128, 128, 256))
    t4k, cb4k = ref.cost_total(path, 8192, 28672, 4096, (128, 128, 256))
    assert not cb16 and cb4k

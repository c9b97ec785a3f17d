"""GPU parity: the sm_100a kernels (through the C ABI in liblqg.so) against the
CPU oracle and the reference's golden vectors. Bar (BASELINE.json north_star):
INT32 accumulators and dequantized INT8 weights bit-exact; F32 output
bit-identical to the reference epilogue (quant.cpp:125-127); F16/BF16 equal to
round-to-nearest-even of that F32 (so <= 1e-3 of max|Y| for F16, <= 1 BF16 ulp)."""
import os

import numpy as np
import pytest

from conftest import make_acts, make_weights

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "the gpu suite needs a B200"
    return torch


def to_bundle(lqg, b: dict):
    return lqg.QuantizedWeightBundle(b["n"], b["k"], b["group_size"], lqg.WeightLayout(b["layout"]),
                                     lqg.FragmentDescriptor(), b["packed"], b["scales"],
                                     b["offsets"], b["channel_scales"])


def check_outputs(torch, dw, q, ts, acc_ref, y_ref):
    xq = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    tsd = torch.from_numpy(np.ascontiguousarray(ts)).cuda()
    acc = dw.gemm_accum(xq).cpu().numpy()
    np.testing.assert_array_equal(acc.astype(np.int64), acc_ref.astype(np.int64))
    y = dw.gemm(xq, tsd, out_dtype=torch.float32).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), y_ref.view(np.uint32))
    for dt in (torch.float16, torch.bfloat16):
        yl = dw.gemm(xq, tsd, out_dtype=dt).cpu()
        assert torch.equal(yl, torch.from_numpy(y_ref).to(dt))
    # F16 tolerance as stated in the north star (implied by the equality above)
    yh = dw.gemm(xq, tsd, out_dtype=torch.float16).float().cpu().numpy()
    assert np.abs(yh - y_ref).max() <= 1e-3 * max(np.abs(y_ref).max(), 1e-30)


SHAPES = [  # m, n, k, g
    (1, 128, 128, 128), (16, 128, 256, 128), (16, 256, 4096, 128), (5, 64, 64, 64),
    (33, 192, 384, 64), (100, 320, 512, 32), (257, 128, 256, 128), (300, 384, 640, 128),
    (1, 4096, 4096, 128), (16, 4096, 4096, 128), (64, 1024, 2048, 256), (129, 256, 768, 128),
    (193, 128, 512, 64), (520, 256, 1024, 128), (7, 100, 96, 32), (2, 1, 256, 64),
]


@pytest.mark.parametrize("m,n,k,g", SHAPES)
def test_accum_and_outputs_bit_exact(torch_cuda, lqg, port, m, n, k, g):
    rng = np.random.default_rng(1000 + m + n + k + g)
    b = port.build_bundle_plain(make_weights(rng, n, k), g)
    q, ts = port.quantize_activations(make_acts(rng, m, k))
    w_i8 = port.bundle_int8(b)
    acc_ref, y_ref = port.gemm_oracle(q, ts, w_i8, b["channel_scales"])
    dw = lqg.DeviceWeights.from_bundle(to_bundle(lqg, b), 0)
    check_outputs(torch_cuda, dw, q, ts, acc_ref, y_ref)
    np.testing.assert_array_equal(dw.dequant().cpu().numpy(), w_i8)


def test_golden_cases_through_reference_api(torch_cuda, lqg):
    """The reference's own outputs (tests/golden/gemm.npz) reproduced through the
    drop-in mirror of lq::gemm_w4a8_accum / lq::gemm_w4a8, both layouts, both
    engines, the reference tile configs."""
    d = np.load(os.path.join(GOLD, "gemm.npz"))
    for ci in range(int(d["n_cases"])):
        m, n, k, g, layout = d[f"c{ci}_dims"].tolist()
        b = lqg.QuantizedWeightBundle(n, k, g, lqg.WeightLayout(layout), lqg.FragmentDescriptor(),
                                      d[f"c{ci}_packed"], d[f"c{ci}_scales"], d[f"c{ci}_offsets"],
                                      d[f"c{ci}_channel_scales"])
        act = lqg.ActivationQuant(m, k, d[f"c{ci}_q"].reshape(-1), d[f"c{ci}_ts"])
        engines = [lqg.Engine.Scalar]
        if n % 64 == 0 and k % 64 == 0 and g % 64 == 0:
            engines.append(lqg.Engine.Packed)
        for e in engines:
            for tile in (lqg.TileConfig(), lqg.TileConfig(32, 128, 128), lqg.TileConfig(16, 256, 192)):
                acc = lqg.gemm_w4a8_accum(act, b, tile, e)
                np.testing.assert_array_equal(acc, d[f"c{ci}_acc"].reshape(-1), err_msg=f"case {ci}")
            y = lqg.gemm_w4a8(act, b, lqg.TileConfig(), e)
            np.testing.assert_array_equal(y.view(np.uint32), d[f"c{ci}_y"].reshape(-1).view(np.uint32))
        if f"c{ci}_w_i8" in d:
            np.testing.assert_array_equal(b.device_weights(0).dequant().cpu().numpy(), d[f"c{ci}_w_i8"])


def test_known_answers(torch_cuda, lqg):
    """test_gemm.cpp:29-92: constant row -> 127*119; one-hot rows read back W^;
    zero activations -> exactly zero."""
    d = np.load(os.path.join(GOLD, "known.npz"))
    b = lqg.QuantizedWeightBundle(1, 64, 64, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                  d["const_packed"], d["const_scales"], d["const_offsets"],
                                  d["const_channel_scales"])
    assert b.scale_of(0, 0) == 1 and b.offset_of(0, 0) == 247
    act = lqg.ActivationQuant(1, 64, d["const_q"].reshape(-1), d["const_ts"])
    assert lqg.gemm_w4a8_accum(act, b, lqg.TileConfig(), lqg.Engine.Scalar)[0] == 127 * 119
    y = lqg.gemm_w4a8(act, b, lqg.TileConfig(), lqg.Engine.Scalar)
    assert y[0] == d["const_y"][0, 0] and abs(y[0] - 60.0) < 60.0 * 1e-5
    ob = lqg.QuantizedWeightBundle(64, 128, 64, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                   d["onehot_packed"], d["onehot_scales"], d["onehot_offsets"],
                                   d["onehot_channel_scales"])
    act = lqg.ActivationQuant(128, 128, np.eye(128, dtype=np.int8).reshape(-1), np.ones(128, np.float32))
    for e in (lqg.Engine.Scalar, lqg.Engine.Packed):
        acc = lqg.gemm_w4a8_accum(act, ob, lqg.TileConfig(), e).reshape(128, 64)
        np.testing.assert_array_equal(acc, d["onehot_w_i8"].T.astype(np.int32))
    zero = lqg.ActivationQuant(4, 128, np.zeros(4 * 128, np.int8), np.ones(4, np.float32))
    assert not lqg.gemm_w4a8(zero, ob).any()


def test_gpu_weight_quantizer_bit_exact(torch_cuda, lqg, port):
    """lqg_weights_quantize (device build_bundle) == the reference quantizer:
    codes, group scales/offsets, channel scales, incl. golden edge rows."""
    torch = torch_cuda
    d = np.load(os.path.join(GOLD, "quant.npz"))
    cases = [(d[f"q{ci}_w"], int(d[f"q{ci}_g"])) for ci in range(int(d["n_cases"]))]
    rng = np.random.default_rng(5)
    cases.append((make_weights(rng, 300, 1024), 128))
    cases.append((make_weights(rng, 130, 768, std=3.0), 256))
    for w, g in cases:
        dw = lqg.DeviceWeights.quantize(torch.from_numpy(w).cuda(), g)
        e = dw.export()
        b = port.build_bundle_plain(w, g)
        np.testing.assert_array_equal(e.packed_weights, b["packed"])
        np.testing.assert_array_equal(e.group_scales, b["scales"])
        np.testing.assert_array_equal(e.group_offsets, b["offsets"])
        np.testing.assert_array_equal(e.channel_scales.view(np.uint32), b["channel_scales"].view(np.uint32))
        np.testing.assert_array_equal(dw.dequant().cpu().numpy(), port.bundle_int8(b))
    bad = torch.zeros(2, 64, device="cuda")
    bad[1, 5] = float("nan")
    with pytest.raises(lqg.ValidationError, match=r"non-finite weight at \(1, 5\)"):
        lqg.DeviceWeights.quantize(bad, 64)


def test_gpu_activation_quantizer_bit_exact(torch_cuda, lqg, port):
    """lqg_quantize_activations == quantize_activations_per_token (gemm.cpp:19-47)."""
    torch = torch_cuda
    d = np.load(os.path.join(GOLD, "act.npz"))
    xs = [d[f"a{i}_x"] for i in range(int(d["n_cases"]))]
    xs.append(make_acts(np.random.default_rng(3), 33, 4096))
    for x in xs:
        q, ts = lqg.quantize_activations(torch.from_numpy(x).cuda())
        q0, ts0 = port.quantize_activations(x)
        np.testing.assert_array_equal(q.cpu().numpy(), q0)
        np.testing.assert_array_equal(ts.cpu().numpy().view(np.uint32), ts0.view(np.uint32))
    act = lqg.quantize_activations_per_token(d["a0_x"].reshape(-1), 2, 2)
    assert act.values.tolist() == [64, -127, 0, 0] and act.token_scales[1] == 1.0
    x = np.ones(4, np.float32)
    x[1] = np.inf
    with pytest.raises(lqg.ValidationError, match=r"\(0, 1\)"):
        lqg.quantize_activations_per_token(x, 2, 2)
    with pytest.raises(lqg.ValidationError):
        lqg.quantize_activations_per_token(np.ones(4, np.float32), 3, 2)


def test_exhaustive_lane_box_through_device_dequant(torch_cuda, lqg, port):
    """All 16 x 16 x 239 (code, s, a) lane points (test_quant.cpp:101-117) through
    the mainloop's LQQ routine (lqg_dequant_weights); the 32-bit IMAD carries of
    unreachable combinations also match the reference's packed path."""
    d = np.load(os.path.join(GOLD, "lanes.npz"))
    box = d["box_lo_lane0"]
    pairs = [(s, a) for s in range(1, 17) for a in range(9, 248)]
    n, k, g = len(pairs), 32, 32
    codes = np.tile(np.concatenate([np.arange(16), np.arange(16)[::-1]]).astype(np.uint8), (n, 1))
    b = lqg.QuantizedWeightBundle(n, k, g, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                  port.pack_plain(codes), np.array([p[0] for p in pairs], np.uint8),
                                  np.array([p[1] for p in pairs], np.uint8), np.ones(n, np.float32))
    w8 = lqg.DeviceWeights.from_bundle(b, 0).dequant().cpu().numpy().view(np.uint8)
    for r, (s, a) in enumerate(pairs):
        # lane 0 of each word holds codes 0 / 4 / 8 / 12 ... (k offsets 8w)
        for c in range(16):
            ok = c * s + a <= 255
            got = w8[r, c]
            if ok:
                assert got == (port.dequantize_scalar(c, s, a) & 0xFF)
            if c in (0, 8):  # lane 0 of a word: no incoming carry -> equals the reference box
                assert got == box[c, s - 1, a - 9]
        # whole-word check against the reference packed arithmetic (carries included)
        for wi in range(4):
            el = codes[r, 8 * wi:8 * wi + 8]
            word = port.pack_interleaved(el)
            lo, hi, _ = port.dequant_word(word, s, a)
            want = np.frombuffer(np.array([lo, hi], np.uint32).tobytes(), np.uint8)
            np.testing.assert_array_equal(w8[r, 8 * wi:8 * wi + 8], want)


def test_accumulator_range_guard_and_depth_check(torch_cuda, lqg):
    """gemm.cpp:53-57 / test_gemm.cpp:198-226: k = 133120 accepted, 133184 rejected;
    mismatched depth rejected (test_gemm.cpp:228-234)."""
    def make(k):
        return lqg.QuantizedWeightBundle(1, k, 64, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                         np.zeros(k // 2, np.uint8), np.ones(k // 64, np.uint8),
                                         np.full(k // 64, 128, np.uint8), np.ones(1, np.float32))

    def act(k):
        return lqg.ActivationQuant(1, k, np.zeros(k, np.int8), np.ones(1, np.float32))

    assert lqg.gemm_w4a8_accum(act(133120), make(133120), lqg.TileConfig(), lqg.Engine.Scalar)[0] == 0
    with pytest.raises(lqg.ValidationError, match="accumulator overflow"):
        lqg.gemm_w4a8_accum(act(133184), make(133184), lqg.TileConfig(), lqg.Engine.Scalar)
    with pytest.raises(lqg.ValidationError, match="does not match"):
        lqg.gemm_w4a8_accum(act(64), make(128), lqg.TileConfig(), lqg.Engine.Scalar)
    with pytest.raises(lqg.ValidationError, match="multiple of"):
        lqg.gemm_w4a8_accum(act(128), make(128), lqg.TileConfig(64, 64, 32), lqg.Engine.Packed)


def test_max_depth_extreme_values(torch_cuda, lqg, port):
    """k near the guard with extreme codes: INT32 accumulation stays exact."""
    torch = torch_cuda
    k = 133120
    q = np.full((2, k), 127, np.int8)
    q[1] = -127
    w8_row = np.full(k, 127, np.int64)
    codes = np.full((1, k), 15, np.uint8)
    b = lqg.QuantizedWeightBundle(1, k, 64, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                  port.pack_plain(codes), np.full(k // 64, 8, np.uint8),
                                  np.full(k // 64, 135, np.uint8), np.ones(1, np.float32))
    # 15*8 + 135 - 128 = 127 everywhere
    dw = lqg.DeviceWeights.from_bundle(b, 0)
    acc = dw.gemm_accum(torch.from_numpy(q).cuda()).cpu().numpy()
    assert acc[0, 0] == 127 * 127 * k and acc[1, 0] == -127 * 127 * k
    assert int(w8_row.sum()) * 127 == acc[0, 0]


@pytest.mark.parametrize("n,k,m", [(8192, 28672, 16), (8192, 28672, 4096), (28672, 8192, 1),
                                   (10240, 8192, 300), (4096, 11008, 1024)])
def test_llama_shapes_row_subset(torch_cuda, lqg, port, n, k, m):
    """Full LLaMA-2 layer shapes: device-quantized weights, a seeded subset of
    output rows/columns checked bit-exact against the oracle (rows are
    independent, BASELINE.md §3 'parity at large M')."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    w = torch.randn(n, k, generator=g, device="cuda") * 0.02
    dw = lqg.DeviceWeights.quantize(w, 128)
    x = torch.randn(m, k, generator=g, device="cuda")
    q, ts = lqg.quantize_activations(x)
    acc = dw.gemm_accum(q)
    y = dw.gemm(q, ts, out_dtype=torch.float32)
    rng = np.random.default_rng(m)
    rows = np.sort(rng.choice(m, size=min(m, 64), replace=False))
    cols = np.sort(rng.choice(n, size=256, replace=False))
    w8 = dw.dequant()[torch.from_numpy(cols).cuda()].cpu().numpy()
    e = dw.export()
    np.testing.assert_array_equal(
        w8, port.reconstruct_int8(256, k, 128, port.logical_codes(n, k, 0, e.packed_weights)[cols],
                                  e.group_scales.reshape(n, -1)[cols], e.group_offsets.reshape(n, -1)[cols]))
    qs = q.cpu().numpy()[rows]
    acc_ref, y_ref = port.gemm_oracle(qs, ts.cpu().numpy()[rows], w8, e.channel_scales[cols])
    np.testing.assert_array_equal(acc.cpu().numpy()[np.ix_(rows, cols)].astype(np.int64), acc_ref)
    np.testing.assert_array_equal(y.cpu().numpy()[np.ix_(rows, cols)].view(np.uint32), y_ref.view(np.uint32))


LLAMA7B = [("qkv", 12288, 4096), ("o", 4096, 4096), ("gate_up", 22016, 4096), ("down", 4096, 11008)]
LLAMA70B = [("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 28672, 8192), ("down", 8192, 28672)]


@pytest.mark.parametrize("shape", [s[0] for s in LLAMA7B])
def test_llama7b_shapes_bf16_and_acc(torch_cuda, lqg, port, shape):
    """BASELINE configs[1]: every LLaMA-2-7B layer GEMM at M = 1, 16, 128, 256,
    512 and 1024 (bench sweep points; 128-1024 run the auto_tile schedules) -- INT32 accumulators bit-exact, the F32
    output bit-identical and the BF16 output (what the bench times) exactly the
    RNE of the reference F32 on a seeded subset of rows and columns."""
    torch = torch_cuda
    _, n, k = next(s for s in LLAMA7B if s[0] == shape)
    g = torch.Generator(device="cuda").manual_seed(n * 3 + k)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    e = dw.export()
    rng = np.random.default_rng(n)
    cols = np.sort(rng.choice(n, size=192, replace=False))
    w8 = port.reconstruct_int8(len(cols), k, 128, port.logical_codes(n, k, 0, e.packed_weights)[cols],
                               e.group_scales.reshape(n, -1)[cols], e.group_offsets.reshape(n, -1)[cols])
    for m in (1, 16, 128, 256, 512, 1024):
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        acc = dw.gemm_accum(q).cpu().numpy()
        y32 = dw.gemm(q, ts, out_dtype=torch.float32).cpu().numpy()
        y16 = dw.gemm(q, ts, out_dtype=torch.bfloat16)
        rows = np.sort(rng.choice(m, size=min(m, 48), replace=False))
        acc_ref, y_ref = port.gemm_oracle(q.cpu().numpy()[rows], ts.cpu().numpy()[rows], w8, e.channel_scales[cols])
        np.testing.assert_array_equal(acc[np.ix_(rows, cols)].astype(np.int64), acc_ref)
        np.testing.assert_array_equal(y32[np.ix_(rows, cols)].view(np.uint32), y_ref.view(np.uint32))
        assert torch.equal(y16.cpu()[torch.from_numpy(rows)][:, torch.from_numpy(cols)],
                           torch.from_numpy(y_ref).to(torch.bfloat16))


@pytest.mark.parametrize("shape", [s[0] for s in LLAMA7B])
def test_auto_tile_schedules_match_base_rule(torch_cuda, lqg, shape):
    """The auto_tile corrections (pick_tiles: no pairs for short k, smaller
    token tiles to fill the units, whole tiles instead of split halves,
    32-token tiles for small weights) only
    move the schedule: full INT32 and BF16 outputs equal the base rule's
    (auto_tile=0) at every M where they change it."""
    torch = torch_cuda
    _, n, k = next(s for s in LLAMA7B if s[0] == shape)
    g = torch.Generator(device="cuda").manual_seed(n + k)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    for m in (48, 64, 96, 128, 256, 384, 512, 768, 1024):
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        acc1, y1 = dw.gemm_accum(q), dw.gemm(q, ts)
        with lqg.lq.tune(auto_tile=0):
            acc0, y0 = dw.gemm_accum(q), dw.gemm(q, ts)
        assert torch.equal(acc0, acc1) and torch.equal(y0, y1), m


@pytest.mark.parametrize("m", [16, 4096])
def test_llama70b_bf16_at_bench_shapes(torch_cuda, lqg, port, m):
    """The BF16 outputs the bench times, full LLaMA-2-70B shapes: RNE of the
    reference F32 epilogue (quant.cpp:125-127) on a seeded row/column subset."""
    torch = torch_cuda
    for name, n, k in LLAMA70B:
        g = torch.Generator(device="cuda").manual_seed(n + 2 * k + m)
        dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        y16 = dw.gemm(q, ts)
        e = dw.export()
        rng = np.random.default_rng(n + m)
        cols = np.sort(rng.choice(n, size=96, replace=False))
        rows = np.sort(rng.choice(m, size=min(m, 32), replace=False))
        w8 = port.reconstruct_int8(len(cols), k, 128, port.logical_codes(n, k, 0, e.packed_weights)[cols],
                                   e.group_scales.reshape(n, -1)[cols], e.group_offsets.reshape(n, -1)[cols])
        _, y_ref = port.gemm_oracle(q.cpu().numpy()[rows], ts.cpu().numpy()[rows], w8, e.channel_scales[cols])
        got = y16.cpu()[torch.from_numpy(rows)][:, torch.from_numpy(cols)]
        assert torch.equal(got, torch.from_numpy(y_ref).to(torch.bfloat16)), name
        del dw


def test_one_handle_two_streams_default_workspaces(torch_cuda, lqg):
    """The boundary's re-entrancy contract: one immutable
    handle launched concurrently on two streams without explicit workspaces
    (each stream gets its own default split-K workspace) -- every result is
    bit-identical to the serial one."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(5)
    dw = lqg.DeviceWeights.quantize(torch.randn(8192, 8192, generator=g, device="cuda") * 0.02, 128)
    inputs = [lqg.quantize_activations(torch.randn(m, 8192, generator=g, device="cuda")) for m in (1, 16, 77, 200, 513)]
    want = [(dw.gemm_accum(q), dw.gemm(q, ts)) for q, ts in inputs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    got = []
    for rep in range(6):
        for i, (q, ts) in enumerate(inputs):
            st = streams[(i + rep) % 2]
            with torch.cuda.stream(st):
                got.append((i, dw.gemm_accum(q, stream=st), dw.gemm(q, ts, stream=st)))
    torch.cuda.synchronize()
    for i, a, y in got:
        assert torch.equal(a, want[i][0]) and torch.equal(y, want[i][1]), i


def test_host_call_is_reentrant_across_threads(torch_cuda, lqg):
    """lqg_gemm_w4a8_host from four host threads on one handle at once
    (pooled staging contexts, no shared mutable state): bit-identical to the
    serial calls."""
    import threading
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(6)
    dw = lqg.DeviceWeights.quantize(torch.randn(4096, 4096, generator=g, device="cuda") * 0.02, 128)
    work = []
    for m in (1, 33, 256, 2100):
        q, ts = lqg.quantize_activations(torch.randn(m, 4096, generator=g, device="cuda"))
        qh, th = q.cpu().pin_memory(), ts.cpu().pin_memory()
        ref = torch.empty(m, 4096, dtype=torch.bfloat16).pin_memory()
        dw.gemm_host(qh, th, ref)
        work.append((qh, th, ref))
    errors = []

    def worker(tid):
        try:
            for rep in range(8):
                qh, th, ref = work[(tid + rep) % len(work)]
                y = torch.empty_like(ref).pin_memory()
                dw.gemm_host(qh, th, y)
                if not torch.equal(y, ref):
                    errors.append((tid, rep))
        except Exception as exc:  # surfaced below
            errors.append(repr(exc))

    th_ = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in th_:
        t.start()
    for t in th_:
        t.join()
    assert not errors, errors


def test_device_api_validates_scales_and_outputs(torch_cuda, lqg):
    """ts / out of the wrong dtype, device or shape are rejected before the
    launch (no out-of-bounds writes, no sticky context errors)."""
    torch = torch_cuda
    dw = lqg.DeviceWeights.quantize(torch.randn(256, 512, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(8, 512, device="cuda"))
    with pytest.raises(lqg.ValidationError):
        dw.gemm(q, ts.cpu())
    with pytest.raises(lqg.ValidationError):
        dw.gemm(q, ts.double())
    with pytest.raises(lqg.ValidationError):
        dw.gemm(q, ts[:4])
    with pytest.raises(lqg.ValidationError):
        dw.gemm(q, ts, out=torch.empty(4, 256, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(lqg.ValidationError):
        dw.gemm(q, ts, out=torch.empty(8, 256, dtype=torch.int8, device="cuda"))
    with pytest.raises(lqg.ValidationError):
        dw.gemm_accum(q, out=torch.empty(8, 256, dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(dw.gemm(q, ts), dw.gemm(q, ts))


def test_bundle_mutation_is_seen_by_the_mirror(torch_cuda, lqg, port):
    """The reference re-reads the bundle on every call; so does the mirror:
    changing a bundle's arrays after a GEMM changes the next GEMM's result."""
    rng = np.random.default_rng(9)
    n, k = 128, 256
    b = port.build_bundle_plain(make_weights(rng, n, k), 128)
    bundle = lqg.QuantizedWeightBundle(n, k, 128, lqg.WeightLayout.PlainRowMajor, lqg.FragmentDescriptor(),
                                       b["packed"].copy(), b["scales"].copy(), b["offsets"].copy(),
                                       b["channel_scales"].copy())
    q, ts = port.quantize_activations(make_acts(rng, 4, k))
    act = lqg.ActivationQuant(4, k, q.reshape(-1), ts)
    y1 = lqg.gemm_w4a8(act, bundle)
    bundle.channel_scales = bundle.channel_scales * 2
    y2 = lqg.gemm_w4a8(act, bundle)
    b2 = dict(b, channel_scales=bundle.channel_scales)
    _, y_ref = port.gemm_oracle(q, ts, port.bundle_int8(b2), b2["channel_scales"])
    np.testing.assert_array_equal(y2.reshape(4, n).view(np.uint32), y_ref.view(np.uint32))
    assert not np.array_equal(y1, y2)


def test_linearity_determinism_and_split_k(torch_cuda, lqg):
    """Size-independent properties at full scale: doubling the activation codes
    doubles the accumulators exactly (test_gemm.cpp:152-172); repeated launches
    (stream-K split tiles reduced in a different order each time) are
    bit-identical."""
    torch = torch_cuda
    n, k = 8192, 28672
    g = torch.Generator(device="cuda").manual_seed(1)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    for m in (1, 16, 77, 2048):
        q = torch.randint(-63, 64, (m, k), generator=g, device="cuda", dtype=torch.int8)
        a1 = dw.gemm_accum(q)
        a2 = dw.gemm_accum(q * 2)
        assert torch.equal(a2, a1 * 2)
        for _ in range(3):
            assert torch.equal(dw.gemm_accum(q), a1)


def test_concurrent_streams_with_own_workspaces(torch_cuda, lqg):
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(2)
    dw = lqg.DeviceWeights.quantize(torch.randn(4096, 4096, generator=g, device="cuda") * 0.02, 128)
    qs = [torch.randint(-127, 128, (m, 4096), generator=g, device="cuda", dtype=torch.int8)
          for m in (16, 48)]
    ref = [dw.gemm_accum(q) for q in qs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    wss = [lqg.Workspace(0), lqg.Workspace(0)]
    outs = [None, None]
    torch.cuda.synchronize()
    for _ in range(5):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                outs[i] = dw.gemm_accum(qs[i], workspace=wss[i], stream=streams[i])
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(outs[i], ref[i])


def test_host_call_cached_image_and_pitches(torch_cuda, lqg, port):
    """lqg_gemm_w4a8_host == device path; a prepacked image (offline cache)
    uploads to the same results; ldx > k and ldy > n (writing a column slice of a
    wider buffer, as the N-split gather does)."""
    torch = torch_cuda
    rng = np.random.default_rng(9)
    n, k, m = 320, 1024, 21
    b = to_bundle(lqg, port.build_bundle_plain(make_weights(rng, n, k), 128))
    q, ts = port.quantize_activations(make_acts(rng, m, k))
    acc_ref, y_ref = port.gemm_oracle(q, ts, port.bundle_int8(dict(
        n=n, k=k, group_size=128, layout=0, packed=b.packed_weights, scales=b.group_scales,
        offsets=b.group_offsets, channel_scales=b.channel_scales)), b.channel_scales)
    dw = lqg.DeviceWeights.from_image(b.prepack(), b.channel_scales, n, k, 128, 0)
    xh = torch.from_numpy(q).pin_memory()
    th = torch.from_numpy(ts).pin_memory()
    yh = torch.empty(m, n, dtype=torch.float32).pin_memory()
    dw.gemm_host(xh, th, yh)
    np.testing.assert_array_equal(yh.numpy().view(np.uint32), y_ref.view(np.uint32))
    xw = torch.zeros(m, k + 64, dtype=torch.int8, device="cuda")
    xw[:, :k] = torch.from_numpy(q).cuda()
    yw = torch.full((m, n + 96), 7.0, dtype=torch.float32, device="cuda")
    dw.gemm(xw[:, :k], torch.from_numpy(ts).cuda(), out=yw[:, 32:32 + n])
    np.testing.assert_array_equal(yw[:, 32:32 + n].cpu().numpy().view(np.uint32), y_ref.view(np.uint32))
    assert (yw[:, :32] == 7).all() and (yw[:, 32 + n:] == 7).all()


def test_launch_counter_counts_native_kernels(torch_cuda, lqg):
    torch = torch_cuda
    dw = lqg.DeviceWeights.quantize(torch.randn(256, 256, device="cuda"), 128)
    q, ts = lqg.quantize_activations(torch.randn(4, 256, device="cuda"))
    c0 = lqg.launch_count()
    dw.gemm(q, ts)
    dw.gemm_accum(q)
    assert lqg.launch_count() - c0 == 2


def test_reference_acceptance_gate_through_cpp_dropin(torch_cuda):
    """The reference's own acceptance criterion 6 (acceptance.cpp:265-315: 100
    random GEMMs, both engines, both layouts, three tile configs, bit-exact vs
    the int64 oracle, F32 within 1e-6) with lq::gemm_w4a8[_accum] provided by
    integration/lq_gemm_lqg.cpp over the lqg C ABI (built by oracle/Makefile
    `dropin` from the reference sources into oracle/_ref/)."""
    import subprocess
    binary = os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref", "acceptance_lqg")
    if not os.path.exists(binary):
        pytest.skip("oracle/_ref/acceptance_lqg not built (reference sources absent)")
    r = subprocess.run([binary, "--criterion", "6"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[PASS] criterion 6" in r.stdout, r.stdout


@pytest.mark.parametrize("m", [2048, 3001, 9000])
def test_host_call_pipelined_chunks(torch_cuda, lqg, m):
    """lqg_gemm_w4a8_host cuts large calls into row chunks pipelined over
    copy-in / GEMM / copy-out streams; the result must equal the single device
    launch byte for byte (pinned and pageable host buffers, accumulators too)."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(m)
    n, k = 384, 640
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
    y_dev = dw.gemm(q, ts).cpu()
    for pin in (True, False):
        qh, th = q.cpu(), ts.cpu()
        yh = torch.empty(m, n, dtype=torch.bfloat16)
        if pin:
            qh, th, yh = qh.pin_memory(), th.pin_memory(), yh.pin_memory()
        dw.gemm_host(qh, th, yh)
        assert torch.equal(yh, y_dev)
    acc_h = np.zeros((m, n), np.int32)
    lqg._lib.lib().lqg_gemm_w4a8_accum_host(dw.handle, q.cpu().numpy().ctypes.data, m,
                                            acc_h.ctypes.data, None)
    np.testing.assert_array_equal(acc_h, dw.gemm_accum(q).cpu().numpy())


def test_fanout_epilogue_writes_every_destination(torch_cuda, lqg):
    """lqg_gemm_w4a8_fanout (the fused all-gather building block of the N-split
    driver): every destination -- here column slices of several full-width
    buffers on this GPU, standing in for the peers' Y over NVLink -- receives
    exactly the lqg_gemm_w4a8 output; columns outside the slice stay untouched."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(5)
    n_full, k, m = 1024, 768, 300
    s, e = 256, 640
    dw = lqg.DeviceWeights.quantize(torch.randn(e - s, k, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
    ref = dw.gemm(q, ts)
    bufs = [torch.full((m, n_full), 7.0, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
    dw.gemm_fanout(q, ts, [b[:, s:e] for b in bufs])
    for b in bufs:
        assert torch.equal(b[:, s:e], ref)
        assert bool((b[:, :s] == 7).all()) and bool((b[:, e:] == 7).all())
    with pytest.raises(lqg.ValidationError):
        dw.gemm_fanout(q, ts, [bufs[0][:, s:e], bufs[1][:, s:e - 1]])


def test_column_parallel_p2p_single_rank(torch_cuda, lqg):
    """tp.ColumnParallelW4A8(gather='p2p') on one rank: symmetric-memory output
    written by the fan-out epilogue equals the plain GEMM."""
    torch = torch_cuda
    from paper_2509_01229_b200 import tp
    g = torch.Generator(device="cuda").manual_seed(6)
    n, k, m = 512, 1024, 40
    w = torch.randn(n, k, generator=g, device="cuda") * 0.02
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
    layer = tp.ColumnParallelW4A8.from_weights(w, 128, 0, 1)
    layer.gather = "p2p"
    try:
        y = layer(q, ts)
    except Exception as exc:  # symmetric memory needs a distributed backend on some builds
        pytest.skip(f"symmetric memory unavailable: {exc}")
    assert torch.equal(y, layer.dw.gemm(q, ts))


def _with_tune(lqg, fn, **knobs):
    with lqg.lq.tune(**knobs):
        return fn()


@pytest.mark.parametrize("m,n,k", [(400, 256, 1024), (1000, 2048, 4096), (4096, 1024, 8192), (300, 384, 640),
                                   (8192, 512, 1024), (333, 8192, 1024)])
def test_cta_pair_mode_matches(torch_cuda, lqg, m, n, k):
    """CTA-pair kernel (cluster of two, tcgen05 cta_group::2, M = 256, each
    CTA loading half of every activation tile; the default from 48 tokens)
    is bit-identical to the one-CTA kernel (tune pair=0), accumulators and BF16."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(m + n)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))

    def run():
        r = dw.gemm_accum(q), dw.gemm(q, ts)
        torch.cuda.synchronize()
        return r
    acc0, y0 = _with_tune(lqg, run, pair=0)
    acc1, y1 = _with_tune(lqg, run, pair=1)
    assert torch.equal(acc0, acc1) and torch.equal(y0, y1)


@pytest.mark.parametrize("m,n,k,g", [(320, 256, 512, 128), (517, 512, 768, 64), (1100, 256, 1024, 256)])
def test_cta_pair_mode_matches_oracle(torch_cuda, lqg, port, m, n, k, g):
    """Default-path pair kernel against the CPU oracle (gemm.cpp:225-243,
    quant.cpp:125-127): INT32 bit-exact, F32 bit-identical, ragged token tail."""
    torch = torch_cuda
    rng = np.random.default_rng(m + n + k)
    b = port.build_bundle_plain(make_weights(rng, n, k), g)
    dw = lqg.DeviceWeights.from_bundle(to_bundle(lqg, b), 0)
    q, ts = port.quantize_activations(make_acts(rng, m, k))
    acc_ref, y_ref = port.gemm_oracle(q, ts, port.bundle_int8(b), b["channel_scales"])
    xq, tsd = torch.from_numpy(q).cuda(), torch.from_numpy(ts).cuda()
    acc = _with_tune(lqg, lambda: dw.gemm_accum(xq).cpu().numpy(), pair=1)
    y = _with_tune(lqg, lambda: dw.gemm(xq, tsd, out_dtype=torch.float32).cpu().numpy(), pair=1)
    np.testing.assert_array_equal(acc.astype(np.int64), acc_ref)
    np.testing.assert_array_equal(y.view(np.uint32), y_ref.view(np.uint32))


def test_pair_threshold_boundary_is_seamless(torch_cuda, lqg):
    """m = 47 (one-CTA kernel) and m = 48 (pair kernel by default) agree on
    their common rows: the automatic switch never changes results."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(319)
    dw = lqg.DeviceWeights.quantize(torch.randn(1024, 2048, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(48, 2048, generator=g, device="cuda"))
    a319, y319 = dw.gemm_accum(q[:47]), dw.gemm(q[:47], ts[:47])
    a320, y320 = dw.gemm_accum(q), dw.gemm(q, ts)
    assert torch.equal(a319, a320[:47]) and torch.equal(y319, y320[:47])


@pytest.mark.parametrize("m,n,k", [(1, 640, 2304), (16, 1024, 4096), (48, 512, 1280), (130, 768, 2048),
                                   (200, 256, 8192), (700, 512, 1536)])
@pytest.mark.parametrize("knobs", [dict(max_w_stages=2), dict(max_w_stages=4, x_ring_bytes=1024),
                                   dict(max_x_stages=2, x_ring_bytes=1024), dict(grid=7), dict(grid=64, no_dp=1),
                                   dict(max_bn=32), dict(pair=1, pair_single_tile=1), dict(no_pdl=1),
                                   dict(acc_stages=1)])
def test_schedule_knobs_bit_exact(torch_cuda, lqg, m, n, k, knobs):
    """Every ring split (2-stage W ring, minimal X ring), grid size, token
    tile and pair policy gives the same INT32 accumulators and BF16 outputs as
    the default schedule: the decoupled W/X rings, the alternating dequant
    warpgroups and the split-K exchange are exercised at their edges."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n + k)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
    acc0, y0 = dw.gemm_accum(q), dw.gemm(q, ts)
    with lqg.tune(**knobs):
        acc1, y1 = dw.gemm_accum(q), dw.gemm(q, ts)
    torch.cuda.synchronize()
    assert torch.equal(acc0, acc1) and torch.equal(y0, y1)


@pytest.mark.parametrize("m", [1, 16, 40, 200])
def test_pdl_launch_chain(torch_cuda, lqg, m):
    """Back-to-back launches on one stream overlap under programmatic
    dependent launch (the next grid streams its first weight chunks before
    griddepcontrol.wait) and share one split-K workspace: a chain over
    alternating weights, shapes and output kinds is bit-identical to the same
    launches each followed by a device synchronize."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(77 + m)
    shapes = [(4096, 4096), (1024, 11008), (12288, 4096), (4096, 4096)]
    dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
           for n, k in shapes]
    xs = {k: lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda")) for _, k in shapes}
    ws = lqg.Workspace(0)

    def chain(sync):
        outs = []
        for rep in range(3):
            for i, dw in enumerate(dws):
                q, ts = xs[dw.k]
                if (i + rep) % 3 == 0:
                    outs.append(dw.gemm_accum(q, workspace=ws))
                else:
                    outs.append(dw.gemm(q, ts, out_dtype=torch.bfloat16 if i % 2 else torch.float32,
                                        workspace=ws))
                if sync:
                    torch.cuda.synchronize()
        torch.cuda.synchronize()
        return outs
    ref = chain(True)
    for _ in range(3):
        for a, b in zip(ref, chain(False)):
            assert torch.equal(a, b)


def test_split_k_sequence_stress(torch_cuda, lqg):
    """Regression for a ring-parity race (odd W rings let one dequant warpgroup
    run two phases ahead of the other and read a weight slot that had not
    landed): the sequence that exposed it -- large-token-tile split-K launches
    of different shapes and kernels back to back on one stream, repeated --
    must give exact INT32 accumulators (checked against an exact float64
    product of the dequantized weights) every time."""
    torch = torch_cuda
    cfgs = [(4096, 1024, 8192), (1000, 2048, 4096), (2048, 384, 640), (3001, 384, 640)]
    data = []
    for (m, n, k) in cfgs:
        g = torch.Generator(device="cuda").manual_seed(m + n)
        dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
        q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
        ref = (q.to(torch.float64) @ dw.dequant().to(torch.float64).T).to(torch.int32)
        data.append((dw, q, ts, ref))
    for _ in range(6):
        for dw, q, ts, ref in data:
            for pair in (0, 1):
                with lqg.tune(pair=pair):
                    acc = dw.gemm_accum(q)
                    dw.gemm(q, ts)
                assert torch.equal(acc, ref)


@pytest.mark.parametrize("m,n,k", [(128, 8192, 2048), (64, 8192, 4096), (128, 4096, 28672), (100, 2048, 2048)])
def test_quad_cluster_split_k_exact(torch_cuda, lqg, m, n, k):
    """Quad mode (tiles split into two halves whose CTA pairs form one 4-CTA
    cluster; the contributor's INT32 partial reaches the finisher through a
    DSMEM bulk copy): exact accumulators against a float64 product of the
    dequantized weights, F32 / BF16 outputs identical to the L2-exchange
    path (no_quad), over repeated back-to-back launches."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n + k)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
    ref = (q.to(torch.float64) @ dw.dequant().to(torch.float64).T).to(torch.int32)
    with lqg.tune(no_quad=1):
        y32 = dw.gemm(q, ts, out_dtype=torch.float32).clone()
        ybf = dw.gemm(q, ts).clone()
    for _ in range(8):
        assert torch.equal(dw.gemm_accum(q), ref)
        assert torch.equal(dw.gemm(q, ts, out_dtype=torch.float32), y32)
        assert torch.equal(dw.gemm(q, ts), ybf)


def test_tune_rejects_unknown_and_out_of_range(lqg):
    with pytest.raises(lqg.ValidationError):
        lqg.tune_set("no_such_knob", 1)
    with pytest.raises(lqg.ValidationError):
        lqg.tune_set("max_w_stages", 1)
    assert lqg.tune_get("pair") == -1


@pytest.mark.parametrize("m,n,k", [(4096, 8192, 8192), (1000, 4096, 4096), (300, 2048, 1024)])
def test_bf16_equals_rne_of_f32_full_output(torch_cuda, lqg, m, n, k):
    """Every BF16 output equals RNE of the F32 output (itself bit-identical to
    the reference epilogue, quant.cpp:125-127) over the full matrix -- at
    4096 x 8192 that includes ~10^4 values within a few float ulps of a BF16
    rounding midpoint, where a single-rounding FP32 shortcut would differ."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    dw = lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128)
    q, ts = lqg.quantize_activations(torch.randn(m, k, generator=g, device="cuda"))
    y32 = dw.gemm(q, ts, out_dtype=torch.float32)
    y16 = dw.gemm(q, ts, out_dtype=torch.bfloat16)
    assert torch.equal(y16, y32.to(torch.bfloat16))


def test_extreme_scales_bit_exact(torch_cuda, lqg, port):
    """Channel and token scales far from the usual range (tiny, huge, zero
    token scales): F32 bit-identical to the reference epilogue, F16/BF16 its
    RNE (F16 overflows to inf exactly where the reference F32 does)."""
    torch = torch_cuda
    rng = np.random.default_rng(77)
    m, n, k, g = 200, 256, 512, 128
    b = port.build_bundle_plain(make_weights(rng, n, k), g)
    cs = b["channel_scales"].copy()
    cs[:6] = [1e-30, 3e-19, 1e20, 2.5e25, 7e-18, 1e18]
    b["channel_scales"] = cs.astype(np.float32)
    q, ts = port.quantize_activations(make_acts(rng, m, k))
    ts = ts.copy()
    ts[[0, 17, 33, 150]] = [0.0, 1e-25, 1e12, 5e9]
    ts = ts.astype(np.float32)
    acc_ref, y_ref = port.gemm_oracle(q, ts, port.bundle_int8(b), b["channel_scales"])
    assert np.isinf(y_ref).any() and (y_ref == 0).any()
    dw = lqg.DeviceWeights.from_bundle(to_bundle(lqg, b), 0)
    xq = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    tsd = torch.from_numpy(np.ascontiguousarray(ts)).cuda()
    np.testing.assert_array_equal(dw.gemm_accum(xq).cpu().numpy().astype(np.int64), acc_ref.astype(np.int64))
    y = dw.gemm(xq, tsd, out_dtype=torch.float32).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), y_ref.view(np.uint32))
    for dt in (torch.float16, torch.bfloat16):
        assert torch.equal(dw.gemm(xq, tsd, out_dtype=dt).cpu(), torch.from_numpy(y_ref).to(dt))

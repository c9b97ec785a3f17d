#!/usr/bin/env python3
"""bench.py — LiquidGEMM W4A8 GEMM on B200 (sm_100a) vs the reference CPU path.

Metric (BASELINE.json): W4A8 GEMM TOPS & %roofline (HBM/INT8) vs M=1..4096,
1/2/4/8 B200 vs CPU ref.

One "step" = one pass of the hot path over the workload: every LLaMA-2-70B
linear-layer shape (qkv 10240x8192, o 8192x8192, gate_up 28672x8192,
down 8192x28672; BASELINE configs[2]) at every M of the sweep
1,2,4,...,4096 — 52 W4A8 GEMMs, group size 128, BF16 output. value = total
INT8 ops of the step / device time (TOPS, whole job). For N>1 the weights are
column-sharded (N-split) across ranks and each GEMM's row output is
all-gathered with NCCL (strong scaling: total work fixed).

  python bench.py [--gpus N --steps K --warmup W] [--impl lqg|reference]
                  [--workload llama2-70b|llama2-7b|mixtral-8x7b] [--no-cpu-baseline]

Inputs are synthetic and resident in HBM before timing; weights are quantized
on the GPU with the reference's two-level LiquidQuant quantizer (bit-exact with
build_bundle, quant.cpp:203-232). L2 hygiene: consecutive launches use
different weights; the step cycles 310 MB of packed weights (> 126 MB L2)
between reuses of any one matrix.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "llama2-70b": dict(
        shapes=[("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 28672, 8192),
                ("down", 8192, 28672)],
        m_sweep=[1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]),
    "llama2-7b": dict(
        shapes=[("qkv", 12288, 4096), ("o", 4096, 4096), ("gate_up", 22016, 4096),
                ("down", 4096, 11008)],
        m_sweep=[1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]),
    "mixtral-8x7b": dict(
        shapes=[("w1w3", 14336, 4096), ("w2", 4096, 14336)],
        m_sweep=[1, 2, 4, 8, 16, 32, 64, 512, 1024, 2048, 4096]),
    "llama2-70b-down": dict(
        shapes=[("down", 8192, 28672)],
        m_sweep=[1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]),
}
GROUP = 128


def load_peaks():
    """Roofline denominators: HBM = MEASURED_PEAKS.json copy bandwidth; INT8 =
    2 x the measured bf16 cuBLAS burst (kind::i8 runs at twice the kind::f16
    rate on sm_100), with the cuBLASLt IMMA burst we measured ourselves
    (profiles/int8_peak.json) reported beside it."""
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)",
             "int8_tops": 2 * 1590.0, "int8_src": "fallback: 2 x bf16 fallback"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        mp = json.load(open(p))
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json copy bandwidth)"
        peaks["int8_tops"] = 2 * float(mp["bf16_tflops"])
        peaks["int8_src"] = "2 x measured bf16 burst (MEASURED_PEAKS.json)"
        if "bf16_tflops_sustained" in mp:
            peaks["int8_tops_sustained"] = 2 * float(mp["bf16_tflops_sustained"])
    p = os.path.join(ROOT, "profiles", "int8_peak.json")
    if os.path.exists(p):
        ip = json.load(open(p))
        peaks["cublaslt_int8_tops"] = float(ip["int8_tops"])
        peaks["cublaslt_int8_tops_sustained"] = float(ip.get("int8_tops_sustained", 0)) or None
        peaks["cublaslt_src"] = "measured cuBLASLt IMMA 8192^3 (profiles/int8_peak.json)"
    return peaks


def algo_bytes(m, n, k, g=GROUP, out_bytes=2):
    """N*K/2 + 2*N*K/g + 4N + M*K + 4M + 2*M*N."""
    return n * k // 2 + 2 * n * k // g + 4 * n + m * k + 4 * m + out_bytes * m * n


def algo_ops(m, n, k):
    return 2 * m * n * k


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml-unavailable"]}
        names = [v for b, v in self.REASONS.items() if self.reasons & b and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference library) — the
# cpu_baseline leg and the --impl reference arm. Never the thing measured for
# our value.
# ---------------------------------------------------------------------------
def cpu_reference_sample(workload: dict, steps: int, warmup: int, threads: int | None = None,
                         bundles=None):
    """Times lq::gemm_w4a8 (Packed engine, DualMmaPacked bundle, TileConfig{64,64,64}) on a
    bounded sample: for each shape, the first 64*T weight rows (one 64-row band per host
    thread) at M in {1, 64, 512}. The reference's cost is linear in M at fixed (N, K)
    (dequant once per tile + M*N*K MACs), and linear in rows at fixed
    threads, so t(shape, M) = (a + b*M) * N / N_sample extrapolates the full sweep.
    T = 1 is the reference as shipped (one call, no threads)."""
    import numpy as np

    import oracle
    if not oracle.ref_available():
        return None, "oracle/_ref/liblqref.so not built"
    ref = oracle.Ref()
    nproc = os.cpu_count() or 1
    min_n = min(n for _, n, _ in workload["shapes"])
    T = threads or max(1, min(nproc, min_n // 64, 128))
    ns = 64 * T
    rng = np.random.default_rng(7)
    ms = [1, 64, 512]
    prepared = []
    for name, n, k in workload["shapes"]:
        if bundles and name in bundles:
            b = bundles[name]
            sub = dict(n=ns, k=k, group_size=GROUP, layout=0,
                       packed=b["packed"][: ns * k // 2], scales=b["scales"][: ns * (k // GROUP)],
                       offsets=b["offsets"][: ns * (k // GROUP)], channel_scales=b["channel_scales"][:ns])
            rb = ref.to_dual(ref.bundle_from_arrays(sub))
        else:
            w = (rng.standard_normal((ns, k)) * 0.02).astype(np.float32)
            rb = ref.build_bundle(w, GROUP, 1)
        sh = ref.shard_prepare(rb, T)
        x = rng.standard_normal((max(ms), k)).astype(np.float32)
        q, ts = ref.quantize_activations(x)
        prepared.append((name, n, k, rb, sh, q, ts))
    times = {}
    for it in range(warmup + steps):
        for name, n, k, rb, sh, q, ts in prepared:
            for m in ms:
                t0 = time.perf_counter()
                ref.gemm_w4a8_sharded(sh, ns, q[:m], ts[:m])
                dt = time.perf_counter() - t0
                if it >= warmup:
                    times.setdefault((name, m), []).append(dt)
    for _, _, _, _, sh, _, _ in prepared:
        ref.shard_free(sh)
    total_t, total_ops, sample_t = 0.0, 0.0, 0.0
    fits = {}
    for name, n, k in workload["shapes"]:
        xs = np.array(ms, float)
        ys = np.array([statistics.median(times[(name, m)]) for m in ms])
        sample_t += ys.sum()
        b, a = np.polyfit(xs, ys, 1)
        a = max(a, 0.0)
        fits[name] = {"a_s": a, "b_s_per_m": b, "rows": ns}
        for m in workload["m_sweep"]:
            total_t += (a + b * m) * n / ns
            total_ops += algo_ops(m, n, k)
    tops = total_ops / total_t / 1e12
    info = {"threads": T, "rows_per_shape": ns, "ms": ms, "fits": fits, "warmup": warmup, "steps": steps,
            "sample_seconds_per_step": sample_t, "predicted_full_sweep_s": total_t}
    return tops, info


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, workload):
    """--impl reference: the unmodified reference lq::gemm_w4a8 (oracle/_ref,
    built from /root/reference/proj/src) on this host's cores; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tops, info = cpu_reference_sample(workload, max(1, args.steps), max(0, args.warmup))
    if tops is None:
        print(json.dumps({"impl": "reference", "unavailable": info}))
        return
    try:
        t1, i1 = cpu_reference_sample(workload, 1, 1, threads=1)
    except Exception as exc:
        t1, i1 = None, repr(exc)
    line = {
        "metric": "W4A8 GEMM TOPS (llama2-70b layer shapes, M sweep 1..4096)",
        "impl": "reference", "value": tops, "unit": "TOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": {"workload": args.workload, "shapes": [[nm, n, k] for nm, n, k in workload["shapes"]],
                   "m_sweep": workload["m_sweep"], "group_size": GROUP, "out_dtype": "f32",
                   "engine": "Packed", "bundle": "DualMmaPacked", "tile": [64, 64, 64]},
        "cpu_baseline": {"value": tops, "unit": "TOPS", "cores": info["threads"],
                         "kind": "reference", "cpu": cpu_model(), "nproc": os.cpu_count(),
                         "sample": f"lq::gemm_w4a8 on rows [0,{info['rows_per_shape']}) of each shape "
                                   f"at M in {info['ms']}, {info['threads']} std::threads (one "
                                   "64-row band each), linear-in-M/linear-in-N extrapolation to "
                                   "the full sweep",
                         "single_thread": {"value": t1, "cores": 1,
                                           "sample": "the reference as shipped (one call, no threads), "
                                                     f"rows [0,{i1['rows_per_shape']}) per shape, same extrapolation"
                                           if t1 else str(i1)}},
        "e2e": {"value": tops, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": info,
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# lqg arm
# ---------------------------------------------------------------------------
def graph_of(fn, torch):
    """CUDA graph of fn() captured on a side stream (None if capture fails,
    e.g. a collective backend that cannot be captured)."""
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    try:
        with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
            fn()
    except Exception as exc:  # fall back to eager, reported in the line
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        return None, repr(exc)[:160]
    torch.cuda.current_stream().wait_stream(st)
    return g, None


def timed_region(run, steps, world, dev, torch, dist, clocks_index=None):
    """Exactly `steps` calls of run() between barrier + synchronize on both
    sides; CUDA events on the launching stream; max over ranks (ms)."""
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(clocks_index) if clocks_index is not None else None
    if clk:
        clk.__enter__()
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, (clk.result() if clk else None)


def run_lqg(args, workload):
    import torch
    import torch.distributed as dist

    import paper_2509_01229_b200 as lqg
    from paper_2509_01229_b200 import tp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        # the driver reads the communicator size from NCCL's init lines
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks = load_peaks()

    shapes = workload["shapes"]
    msweep = workload["m_sweep"]
    mmax = max(msweep)
    gen = torch.Generator(device=dev)

    # ---- weights: N-split shards, quantized on the GPU (LiquidQuant two-level)
    layers = []
    for li, (name, n, k) in enumerate(shapes):
        plan = tp.ShardPlan(n, world, rank, tp.shard_rows(n, world))
        nr = plan.rows[1] - plan.rows[0]
        gen.manual_seed(1234 + 7919 * li + 104729 * rank)
        w = torch.randn(nr, k, generator=gen, device=dev, dtype=torch.float32).mul_(0.02)
        dw = lqg.DeviceWeights.quantize(w, GROUP)
        del w
        L = dict(name=name, n=n, nr=nr, k=k, dw=dw, plan=plan)
        # the GEMM writes its column slice straight into the padded send buffer
        # of the all-gather (output pitch = shard width): no copy, no allocation
        L["send"] = torch.empty(mmax, plan.width, dtype=torch.bfloat16, device=dev)
        if world > 1:
            L["buf"] = torch.empty(world * mmax * plan.width, dtype=torch.bfloat16, device=dev)
            L["yfull"] = torch.empty(mmax, n, dtype=torch.bfloat16, device=dev)
            if args.gather == "p2p":
                L["layer"] = tp.ColumnParallelW4A8(n, k, GROUP, rank, world, device_weights=dw, gather="p2p")
        layers.append(L)
    torch.cuda.synchronize()

    # ---- activations per K, quantized per token on the GPU
    xs = {}
    for k in sorted({k for _, _, k in shapes}):
        gen.manual_seed(99 + k)
        x = torch.randn(mmax, k, generator=gen, device=dev, dtype=torch.float32)
        mask = torch.rand(mmax, k, generator=gen, device=dev) < 1e-3
        x[mask] *= 20
        del mask
        xs[k] = lqg.quantize_activations(x)
        del x
    ws = lqg.Workspace(local)

    def gemm(L, m):
        q, ts = xs[L["k"]]
        L["dw"].gemm(q[:m], ts[:m], out=L["send"][:m, :L["nr"]], workspace=ws)

    def gemm_ag(L, m):
        if world > 1 and args.gather == "p2p":
            q, ts = xs[L["k"]]
            L["layer"](q[:m], ts[:m], out=L["yfull"][:m])
            return
        gemm(L, m)
        if world > 1:
            tp.gather_columns(L["send"][:m], L["plan"], out=L["yfull"][:m], buf=L["buf"])

    def step_gemm_only():
        for m in msweep:
            for L in layers:
                gemm(L, m)

    def step():
        for m in msweep:
            for L in layers:
                gemm_ag(L, m)

    ops_step = sum(algo_ops(m, L["n"], L["k"]) for m in msweep for L in layers)

    # ---- warm-up (eager: kernel attributes, workspaces, NCCL communicators),
    # then CUDA graphs of the step (GEMM + all-gather) and of the GEMMs alone
    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    graph_note = {}
    runs = {}
    for key, fn in (("full", step), ("gemm_only", step_gemm_only)):
        g = None
        if not args.no_graph:
            c0 = lqg.launch_count()
            g, err = graph_of(fn, torch)
            if err:
                graph_note[key] = f"eager (graph capture failed: {err})"
        if g is not None:
            runs[key] = g.replay
            graph_note.setdefault(key, "CUDA graph")
        else:
            runs[key] = fn
            graph_note.setdefault(key, "eager")
        for _ in range(args.warmup):
            runs[key]()
        torch.cuda.synchronize()
    launches_per_step = len(msweep) * len(layers)

    # ---- timed region: exactly K steps between barrier + synchronize
    c0 = lqg.launch_count()
    ms_total, clocks = timed_region(runs["full"], args.steps, world, dev, torch, dist, clocks_index=local)
    host_launches = lqg.launch_count() - c0
    ms_per_step = ms_total / args.steps
    value = ops_step * args.steps / (ms_total * 1e-3) / 1e12
    gpu_launches = launches_per_step * args.steps if graph_note["full"] == "CUDA graph" else host_launches
    gemm_only = None
    if world > 1:
        ms_g, _ = timed_region(runs["gemm_only"], args.steps, world, dev, torch, dist)
        gemm_only = {"value": ops_step * args.steps / (ms_g * 1e-3) / 1e12, "unit": "TOPS",
                     "ms_per_step": ms_g / args.steps, "timing": graph_note["gemm_only"],
                     "note": "same step without the row-output all-gather"}

    # ---- per-M breakdown (graph of R rotations of the layer GEMMs per M)
    sweep, per_shape = [], {}
    if world == 1 and not args.no_sweep:
        sweep, per_shape = run_sweep(layers, msweep, gemm, peaks, torch, local, per_shape_ms=(1, 16))

    # ---- e2e through the reference-facing host-buffer C-ABI call
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, layers, msweep, xs, world, dev, lqg, ops_step)

    # ---- LLaMA-2-7B sweep (BASELINE configs[1]) and MoE grouped (configs[4])
    sweep_7b = moe = None
    if world == 1 and not args.no_sweep and args.workload == "llama2-70b":
        try:
            sweep_7b = run_7b(lqg, dev, peaks, torch)
        except Exception as exc:  # extra evidence must never sink the main number
            sweep_7b = {"error": repr(exc)[:200]}
        try:
            moe = run_moe(lqg, dev, peaks)
        except Exception as exc:
            moe = {"error": repr(exc)[:200]}

    # ---- CPU baseline (rank 0, N=1 only), same warm-up as the reference arm
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(workload)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    def pick(m):
        for r in sweep:
            if r["m"] == m:
                return r
        return None

    roofline = roofline_decode = None
    prof = load_profile_summary()
    big = pick(mmax)
    if big and "power_states" in big:
        ops = sum(algo_ops(mmax, L["n"], L["k"]) for L in layers)
        st = big["power_states"]
        burst = ops / (st["burst"]["us"] * 1e-6) / 1e12
        sust = ops / (st["sustained"]["us"] * 1e-6) / 1e12
        roofline = {"bound": "tensor", "achieved": burst, "peak": peaks["int8_tops"],
                    "unit": "TFLOP/s", "frac": burst / peaks["int8_tops"],
                    "traffic": prof.get("traffic_bytes_M4096"),
                    "at": f"M={mmax}, 4 layer GEMMs, INT8 ops (TOPS), burst: timed 2 s after idle",
                    "peak_src": peaks["int8_src"], "clocks": st["burst"]["clocks"],
                    "vs_cublaslt_int8": {"peak": peaks.get("cublaslt_int8_tops"),
                                         "frac": burst / peaks["cublaslt_int8_tops"] if peaks.get("cublaslt_int8_tops") else None},
                    "sustained": {"achieved": sust, "peak": peaks.get("int8_tops_sustained"),
                                  "frac": sust / peaks["int8_tops_sustained"] if peaks.get("int8_tops_sustained") else None,
                                  "at": "after 6 s of back-to-back replays (power-capped)",
                                  "clocks": st["sustained"]["clocks"]},
                    "sweep_entry": {"achieved": big["tops"], "note": "median of 7 inside the sweep (partly power-capped)"}}
    small = pick(16)
    if small:
        roofline_decode = {"bound": "hbm", "achieved": small["hbm_gbs"], "peak": peaks["hbm_gbs"],
                           "unit": "GB/s", "frac": small["hbm_gbs"] / peaks["hbm_gbs"],
                           "traffic": prof.get("traffic_bytes_M16"),
                           "at": "M=16, 4 layer GEMMs, algorithmic bytes", "peak_src": peaks["hbm_src"],
                           "per_shape": per_shape.get(16), "per_shape_m1": per_shape.get(1)}
    line = {
        "metric": "W4A8 GEMM TOPS (llama2-70b layer shapes, M sweep 1..4096)",
        "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (SURVEY 8d): W~N(0,0.02^2); X~N(0,1) with 0.1% of entries x20; LiquidQuant-quantized on GPU",
        "config": {"workload": args.workload,
                   "shapes": [[nm, n, k] for nm, n, k in shapes], "m_sweep": msweep,
                   "group_size": GROUP, "out_dtype": "bf16", "gemms_per_step": len(msweep) * len(shapes),
                   "parallelism": (f"tp{world} N-split + {args.gather} row-output all-gather" if world > 1 else "single"),
                   "l2": "inputs larger than L2: 310 MB of packed weights cycle between reuses",
                   "timing": graph_note["full"] + "; per-M sweep: median of 7; M <= 64 entries after 1.5 s idle"},
        "gpu_launches": gpu_launches,
        "clocks": clocks,
        "roofline": roofline,
        "roofline_decode": roofline_decode,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gemm_only": gemm_only,
        "sweep": sweep,
        "sweep_llama2_7b": sweep_7b,
        "moe_grouped": moe,
        "peaks": peaks,
    }
    print(json.dumps(line))
    sys.stdout.flush()
    if world > 1:
        dist.destroy_process_group()


def run_sweep(layers, msweep, gemm, peaks, torch, local, per_shape_ms=()):
    """Per-M device time of the layer GEMMs: CUDA graph of R rotations (one
    rotation = every layer once; consecutive launches use different weights),
    median of 7 timings of 3 replays. HBM-bound entries (M <= 64) start after a
    short idle: right after heavy tensor-core work the GPU runs memory-bound
    kernels ~10-30 % slower for about a second (tools/bench_probe.py)."""
    R = 3
    sweep, per_shape = [], {}

    def graph_time(fn, reps=3, n=7):
        g, _ = graph_of(fn, torch)
        g.replay()
        torch.cuda.synchronize()
        samples = []
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1) * 1e-3 / reps)
        return statistics.median(samples), g

    for m in msweep:
        def rot():
            for _ in range(R):
                for L in layers:
                    gemm(L, m)
        if m <= 64:
            time.sleep(1.5)
        t_s, g = graph_time(rot)
        t_s /= R
        states = None
        if m == max(msweep):
            # The tensor-bound entry in both power states (B200 board limit
            # 1000 W: after seconds of back-to-back INT8 MMA the SM clock
            # settles near 1450 MHz, sw_power_cap). Burst: after 2 s idle,
            # 5 replays (~30 ms). Sustained: after 6 s of continuous replays.
            states = {}
            for state, pre in (("burst", 0.0), ("sustained", 6.0)):
                time.sleep(2.0)
                t0 = time.time()
                while time.time() - t0 < pre:
                    for _ in range(10):
                        g.replay()
                    torch.cuda.synchronize()
                with ClockSampler(local, 0.002) as ck:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5):
                        g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                states[state] = {"us": e0.elapsed_time(e1) * 1e-3 / (5 * R) * 1e6, "clocks": ck.result()}
        ops = sum(algo_ops(m, L["n"], L["k"]) for L in layers)
        byts = sum(algo_bytes(m, L["n"], L["k"]) for L in layers)
        entry = {"m": m, "us": t_s * 1e6, "tops": ops / t_s / 1e12, "hbm_gbs": byts / t_s / 1e9,
                 "hbm_frac": byts / t_s / 1e9 / peaks["hbm_gbs"], "int8_frac": ops / t_s / 1e12 / peaks["int8_tops"]}
        if states:
            entry["power_states"] = states
        sweep.append(entry)
        if m in per_shape_ms:
            rows = []
            for L in layers:
                def one(L=L):
                    for _ in range(4):
                        gemm(L, m)
                time.sleep(0.5)
                t1, _ = graph_time(one)
                t1 /= 4
                b1 = algo_bytes(m, L["n"], L["k"])
                rows.append({"shape": L["name"], "n": L["n"], "k": L["k"], "us": t1 * 1e6,
                             "hbm_gbs": b1 / t1 / 1e9, "hbm_frac": b1 / t1 / 1e9 / peaks["hbm_gbs"],
                             "note": "4 back-to-back launches of this shape"})
            per_shape[m] = rows
        del g
    return sweep, per_shape


def run_7b(lqg, dev, peaks, torch):
    """BASELINE configs[1]: the four LLaMA-2-7B linear-layer GEMMs (qkv
    12288x4096, o 4096x4096, gate_up 22016x4096, down 4096x11008) at M = 1..1024:
    graph-amortised device time of the 4-GEMM rotation (3 weight copies per
    shape so consecutive launches miss L2) and the single-launch latency of one
    eager GEMM (host launch + kernel, events around one call after a sync)."""
    wl = WORKLOADS["llama2-7b"]
    g = torch.Generator(device=dev).manual_seed(7)
    copies = 3
    layers = []
    for name, n, k in wl["shapes"]:
        dws = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device=dev) * 0.02, GROUP)
               for _ in range(copies)]
        layers.append(dict(name=name, n=n, k=k, dws=dws,
                           y=torch.empty(max(wl["m_sweep"]), n, dtype=torch.bfloat16, device=dev)))
    xs = {k: lqg.quantize_activations(torch.randn(max(wl["m_sweep"]), k, generator=g, device=dev))
          for k in {k for _, _, k in wl["shapes"]}}
    ws = lqg.Workspace(dev.index or 0)
    out = []
    for m in wl["m_sweep"]:
        def rot():
            for c in range(copies):
                for L in layers:
                    q, ts = xs[L["k"]]
                    L["dws"][c].gemm(q[:m], ts[:m], out=L["y"][:m], workspace=ws)
        if m <= 64:
            time.sleep(1.0)
        gr, _ = graph_of(rot, torch)
        gr.replay()
        torch.cuda.synchronize()
        samples = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1) * 1e-3 / (3 * copies))
        t = statistics.median(samples)
        # single launch: one eager GEMM (down), host launch overhead included
        L = layers[3]
        q, ts = xs[L["k"]]
        qm, tsm, ym, dw0 = q[:m], ts[:m], L["y"][:m], L["dws"][0]
        single = []
        for _ in range(9):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dw0.gemm(qm, tsm, out=ym, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            single.append(e0.elapsed_time(e1) * 1e3)
        ops = sum(algo_ops(m, L["n"], L["k"]) for L in layers)
        byts = sum(algo_bytes(m, L["n"], L["k"]) for L in layers)
        out.append({"m": m, "us_4gemm": t * 1e6, "tops": ops / t / 1e12,
                    "hbm_frac": byts / t / 1e9 / peaks["hbm_gbs"], "int8_frac": ops / t / 1e12 / peaks["int8_tops"],
                    "single_launch_down_us": statistics.median(single)})
        del gr
    return {"shapes": [[nm, n, k] for nm, n, k in wl["shapes"]], "entries": out,
            "timing": "CUDA graph of 3 rotations of the 4 GEMMs (distinct weight copies), median of 7; "
                      "single_launch: one eager lqg_gemm_w4a8 of the down shape, CUDA events around the call"}


def cpu_baseline(workload):
    """The reference's CPU path timed on this host beside the GPU number:
    (ii) one std::thread per 64-row band (nproc threads) and (i) the reference
    as shipped, one thread; both with the reference arm's warm-up."""
    res = {}
    for label, threads in (("threads", None), ("single_thread", 1)):
        try:
            tops, info = cpu_reference_sample(workload, steps=1, warmup=1, threads=threads)
        except Exception as exc:  # baseline must never sink the GPU number
            tops, info = None, f"failed: {exc!r}"
        res[label] = (tops, info)
    tops, info = res["threads"]
    if tops is None:
        return {"value": None, "unit": "TOPS", "cores": 0, "kind": "reference", "sample": f"unavailable: {info}"}
    t1, i1 = res["single_thread"]
    return {"value": tops, "unit": "TOPS", "cores": info["threads"], "kind": "reference",
            "cpu": cpu_model(), "nproc": os.cpu_count(),
            "sample": f"unmodified lq::gemm_w4a8 (oracle/_ref) on rows [0,{info['rows_per_shape']}) of each "
                      f"shape at M in {info['ms']}, {info['threads']} threads (one 64-row band each), 1 warm-up "
                      f"pass, extrapolated linearly in M and N to the full sweep "
                      f"({info['sample_seconds_per_step']:.1f} s of CPU sample)",
            "single_thread": {"value": t1, "unit": "TOPS", "cores": 1,
                              "sample": (f"the reference as shipped (no threads): rows [0,{i1['rows_per_shape']}) "
                                         f"of each shape at M in {i1['ms']}, extrapolated likewise "
                                         f"({i1['sample_seconds_per_step']:.1f} s)") if t1 else str(i1)}}


def run_e2e(args, layers, msweep, xs, world, dev, lqg, ops_step):
    """Same metric through the reference-facing host-buffer call
    (lqg_gemm_w4a8_host): per GEMM, pinned host X/ts -> device, GEMM, device Y ->
    pinned host, synchronous like lq::gemm_w4a8. For N>1: H2D, GEMM on the
    shard, NCCL all-gather, D2H of the full Y."""
    import torch
    import torch.distributed as dist

    from paper_2509_01229_b200 import tp
    mmax = max(msweep)
    hx = {k: (q.cpu().pin_memory(), ts.cpu().pin_memory()) for k, (q, ts) in xs.items()}
    hy = {L["name"]: torch.empty(mmax, L["n"], dtype=torch.bfloat16).pin_memory() for L in layers}
    h2d = sum(m * L["k"] + 4 * m for m in msweep for L in layers)
    d2h = sum(2 * m * L["n"] for m in msweep for L in layers)
    if world > 1:
        dx = {k: (torch.empty_like(q, device=dev), torch.empty_like(ts, device=dev)) for k, (q, ts) in xs.items()}

    def one_step():
        for m in msweep:
            for L in layers:
                qh, th = hx[L["k"]]
                if world == 1:
                    L["dw"].gemm_host(qh[:m], th[:m], hy[L["name"]][:m])
                else:
                    qd, td = dx[L["k"]]
                    qd[:m].copy_(qh[:m], non_blocking=True)
                    td[:m].copy_(th[:m], non_blocking=True)
                    L["dw"].gemm(qd[:m], td[:m], out=L["send"][:m, :L["nr"]])
                    tp.gather_columns(L["send"][:m], L["plan"], out=L["yfull"][:m], buf=L["buf"])
                    hy[L["name"]][:m].copy_(L["yfull"][:m])
                    torch.cuda.synchronize()

    one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": ops_step * steps / dt / 1e12, "unit": "TOPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "path": "lqg_gemm_w4a8_host (C ABI, pinned host buffers)" if world == 1 else
                    "H2D + lqg_gemm_w4a8 + NCCL all-gather + D2H"}


def run_moe(lqg, dev, peaks):
    """BASELINE config 5: Mixtral-8x7B expert FFN GEMMs (w1/w3 14336x4096, w2
    4096x14336; 8 experts, top-2 routing of T tokens, seeded skewed router) as
    ONE grouped launch (lqg_gemm_w4a8_grouped) vs one launch per expert. Device
    time of CUDA-graph replays (8 x 29 MB of weights per GEMM, > L2 with the
    rotation below)."""
    import numpy as np
    import torch
    E = 8
    g = torch.Generator(device=dev)
    g.manual_seed(42)
    experts = {nm: [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device=dev) * 0.02, GROUP)
                    for _ in range(E)] for nm, n, k in (("w1", 14336, 4096), ("w2", 4096, 14336))}
    ws = lqg.Workspace(dev.index or 0)
    rng = np.random.default_rng(0)

    def graph_time(fn, reps=8):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st), torch.cuda.graph(gr, stream=st):
            for _ in range(reps):
                fn()
        torch.cuda.current_stream().wait_stream(st)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    rows_out = []
    for T in (1, 16, 64, 512, 4096):
        p = rng.dirichlet(np.full(E, 2.0))
        ms = np.bincount(rng.choice(E, size=2 * T, p=p), minlength=E).astype(np.uint32).tolist()
        rows = sum(ms)
        for nm, dws in experts.items():
            n, k = dws[0].n, dws[0].k
            xq, ts = lqg.quantize_activations(torch.randn(rows, k, generator=g, device=dev))
            y = torch.empty(rows, n, dtype=torch.bfloat16, device=dev)
            tg = graph_time(lambda: lqg.gemm_grouped(dws, xq, ts, ms, out=y, workspace=ws))

            def per():
                r0 = 0
                for dw, m in zip(dws, ms):
                    if m:
                        dw.gemm(xq[r0:r0 + m], ts[r0:r0 + m], out=y[r0:r0 + m], workspace=ws)
                    r0 += m
            tp_ = graph_time(per)
            used = [m for m in ms if m]
            byts = sum(algo_bytes(m, n, k) for m in used)
            ops = 2 * rows * n * k
            rows_out.append({"tokens": T, "gemm": nm, "experts_m": ms, "grouped_us": tg * 1e6,
                             "per_expert_us": tp_ * 1e6, "grouped_tops": ops / tg / 1e12,
                             "grouped_hbm_frac": byts / tg / 1e9 / peaks["hbm_gbs"],
                             "grouped_int8_frac": ops / tg / 1e12 / peaks["int8_tops"]})
    return rows_out


def load_profile_summary():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def spawn_ranks(args):
    """`--gpus N` without a launcher: re-exec this script under
    torch.distributed.run with N local ranks (one per GPU, NCCL over NVLink)."""
    import socket
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lqg", choices=["lqg", "reference"])
    ap.add_argument("--workload", default="llama2-70b", choices=sorted(WORKLOADS))
    ap.add_argument("--gather", default="nccl", choices=["nccl", "p2p"],
                    help="N>1 row-output all-gather: NCCL collective or fused into the GEMM epilogue")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "lqg":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    run_lqg(args, wl)
    return 0


if __name__ == "__main__":
    sys.exit(main())

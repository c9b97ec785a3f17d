"""The reference's analytic cost model (cost_model.cpp, via oracle/_ref) with
the measured B200 profile (profiles/b200.profile) next to the measured M sweep
of the LLaMA-2-70B 4-layer step (a bench.py JSON line).
  python tools/cost_model.py [profiles/r01_bench.jsonl]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles", "b200.profile")
SHAPES = [(10240, 8192), (8192, 8192), (28672, 8192), (8192, 28672)]


def main():
    ref = oracle.Ref()
    ms, am, ac = ref.profile_diag(PROF)
    print(f"b200 profile: M* = {ms:.1f} (W4A8), alpha*_mem = {am:.3f}, alpha*_comp(150) = {ac:.3f}; "
          f"LiquidQuant alpha = 7/8 = 0.875 ops/element (packed.hpp:89-95)")
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_bench.jsonl")
    line = [l for l in open(path) if l.strip().startswith("{")][-1]
    sweep = {r["m"]: r["us"] for r in json.loads(line)["sweep"]}
    print(f"{'M':>6} {'model_us':>9} {'regime':>8} {'measured_us':>12} {'measured/model':>15}")
    for m in sorted(sweep):
        t, regimes = 0.0, set()
        for n, k in SHAPES:
            s, cb = ref.cost_total(PROF, n, k, m, (128, 128, 256), 7 / 8)
            t += s
            regimes.add("compute" if cb else "memory")
        print(f"{m:6d} {t*1e6:9.1f} {'/'.join(sorted(regimes)):>8} {sweep[m]:12.1f} {sweep[m]/(t*1e6):15.2f}")


if __name__ == "__main__":
    main()

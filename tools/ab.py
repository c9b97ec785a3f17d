"""A/B timing of liblqg variants (or schedule knob sets) in one process per
variant, alternated:
  python tools/ab.py --libs a.so,b.so --ms 16 --rounds 3
  python tools/ab.py --libs a.so --tunes "max_bn=192;max_bn=160" --ms 1024,4096
Times the 70B 4-layer step at each M as a CUDA graph (3 rotations), like bench.py."""
import argparse, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, time
sys.path.insert(0, ROOT)
import torch
import paper_2509_01229_b200 as lqg
for kv in filter(None, TUNE.split(",")):
    kk, vv = kv.split("=")
    lqg.tune_set(kk, int(vv))
shapes = [(10240, 8192), (8192, 8192), (28672, 8192), (8192, 28672)]
ms = MS
g = torch.Generator(device="cuda"); g.manual_seed(1)
layers = [lqg.DeviceWeights.quantize(torch.randn(n, k, generator=g, device="cuda") * 0.02, 128) for n, k in shapes]
xs = {k: lqg.quantize_activations(torch.randn(max(ms), k, generator=g, device="cuda")) for k in (8192, 28672)}
ys = [torch.empty(max(ms), n, dtype=torch.bfloat16, device="cuda") for n, _ in shapes]
ws = lqg.Workspace(0)
out = {}
for m in ms:
    def step():
        for (n, k), dw, y in zip(shapes, layers, ys):
            q, ts = xs[k]
            dw.gemm(q[:m], ts[:m], out=y[:m], workspace=ws)
    step(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        for _ in range(3): step()
    torch.cuda.current_stream().wait_stream(s)
    gr.replay(); torch.cuda.synchronize()
    time.sleep(IDLE)  # burst state: after idle (B200 power-caps within ~1 s of heavy MMA)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): gr.replay()
    e1.record(); torch.cuda.synchronize()
    out[m] = e0.elapsed_time(e1) / 15 * 1e3
print(json.dumps(out))
'''

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--ms", default="16")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--idle", type=float, default=1.5, help="seconds idle before each timing")
    ap.add_argument("--env", default="", help="extra env per lib, ';'-separated list of k=v,k=v")
    ap.add_argument("--tunes", default="", help="';'-separated knob sets k=v,k=v (one variant each)")
    a = ap.parse_args()
    libs = a.libs.split(",")
    tunes = a.tunes.split(";") if a.tunes else [""]
    if len(libs) == 1 and len(tunes) > 1:
        libs = libs * len(tunes)
    if len(tunes) == 1:
        tunes = tunes * len(libs)
    envs = a.env.split(";") if a.env else [""] * len(libs)
    ms = [int(x) for x in a.ms.split(",")]
    res = {i: [] for i in range(len(libs))}
    for r in range(a.rounds):
        for i, lib in enumerate(libs):
            env = dict(os.environ, LQG_LIB_PATH=os.path.abspath(lib))
            for kv in filter(None, envs[i].split(",")):
                k, v = kv.split("=")
                env[k] = v
            code = (CHILD.replace("ROOT", repr(ROOT)).replace("MS", repr(ms)).replace("IDLE", repr(a.idle))
                    .replace("TUNE", repr(tunes[i])))
            o = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            if o.returncode:
                print(lib, "FAILED", o.stderr[-500:]); continue
            res[i].append(json.loads(o.stdout.strip().splitlines()[-1]))
    for i, lib in enumerate(libs):
        for m in ms:
            v = [x[str(m)] for x in res[i]]
            print(f"{os.path.basename(lib):20s} {envs[i] + tunes[i]:30s} M={m:5d}: " + " ".join(f"{t:7.1f}" for t in v) + f"  min {min(v):.1f} us")

if __name__ == "__main__":
    main()

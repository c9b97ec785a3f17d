"""Per-source-line warp-stall samples from an ncu report captured with
--import-source on (the report is read here, no GPU needed):

  python tools/ncu_lines.py gpurun_out/src_10240x8192_m128.ncu-rep [top=30]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
# the header repeats "Source": first is the CUDA line, second the SASS text
idx = {h: i for i, h in enumerate(hdr) if h not in idx} if False else {}
for i, h in enumerate(hdr):
    idx.setdefault(h, i)
samp = idx["Warp Stall Sampling (All Samples)"]
stall_cols = [(h, i) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
file_path = None
for r in rows[hdr_i + 1:]:
    if not r or not r[0]:
        continue
    if r[0] in ("File Path", "Function Name"):
        continue
    try:
        s = float(r[samp])
    except (ValueError, IndexError):
        continue
    st = sorted(((float(r[i]) if r[i] not in ("", "-") else 0.0, h[6:]) for h, i in stall_cols), reverse=True)
    lines.append((s, r[0], r[1][:90], st[:3]))
total = sum(x[0] for x in lines)
print(f"total samples {total:.0f}")
for s, ln, src, st in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / total:5.1f}%  L{ln:>5}  {src:90s}  " + ", ".join(f"{n} {v:.0f}" for v, n in st if v))

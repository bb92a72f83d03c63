"""Top CUDA source lines by warp-stall samples (aggregated over their SASS),
with file:line and the dominant stall reasons.
  python tools/ncu_hot.py <ncu-rep> [N]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
path = "?"
hdr = None
lines = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].strip().isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"])
    except ValueError:
        continue
    stalls = {k[6:]: int(v) for k, v in d.items()
              if k.startswith("stall_") and "Not Issued" not in k and v.strip().isdigit()}
    top = ", ".join(f"{k} {v}" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:3] if v)
    lines.append((s, f"{path}:{r[0]}", r[1].strip()[:90], top))
tot = sum(x[0] for x in lines) or 1
print(f"{len(lines)} source lines, samples {tot}")
for s, loc, src, top in sorted(lines, key=lambda x: -x[0])[:N]:
    print(f"{s:8d} {100 * s / tot:5.1f}%  {loc:22s} {src}  [{top}]")

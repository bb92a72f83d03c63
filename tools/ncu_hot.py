"""Top SASS instructions by warp-stall samples, with CUDA source lines.
  python tools/ncu_hot.py <ncu-rep> [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ni = h.index("Warp Stall Sampling (All Samples)")
si = h.index("Source")
tot = sum((int(r[ni]) if r[ni].strip().isdigit() else 0) for r in data) or 1
print(len(data), "rows, samples", tot)
for r in sorted(data, key=lambda r: -(int(r[ni]) if r[ni].strip().isdigit() else 0))[:N]:
    print(f"{(int(r[ni]) if r[ni].strip().isdigit() else 0):7d} {100 * (int(r[ni]) if r[ni].strip().isdigit() else 0) / tot:5.1f}%  {r[si][:110]}")

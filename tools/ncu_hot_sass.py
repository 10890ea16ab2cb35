"""Top SASS instructions by warp-stall samples from an ncu report
(development): python tools/ncu_hot_sass.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((float(r[si]), idx, r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"{rep}: {int(tot)} samples")
for v, idx, src in sorted(data, reverse=True)[:top]:
    print(f"{v / tot * 100:5.1f}%  #{idx:5d}  {src[:100]}")

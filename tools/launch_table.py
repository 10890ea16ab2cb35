"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per
launch) per kernel as a markdown table; write the top GEMM's DRAM bytes per
launch to profiles/ncu_traffic.json.  usage: python tools/launch_table.py CSV [GZ_OUT]"""
import collections
import csv
import gzip
import json
import shutil
import sys

src = sys.argv[1]
rows = list(csv.reader(open(src)))
start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[start]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per, name = collections.defaultdict(dict), {}
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        v *= 1e-3  # ns -> us
    per[r[ii]][r[mi]] = v
    name[r[ii]] = r[ki]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k, m in per.items():
    short = name[k].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
excl = {"k_fact_error", "k_fact_error_final", "k_gate", "k_symmetrize"}
tot = sum(a[1] for k, a in agg.items() if k not in excl)
print("| kernel | launches | total ms | avg µs | DRAM GB | share of factorization kernels |")
print("|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:18]:
    sh = "—" if k in excl else "%.1f%%" % (100 * a[1] / tot)
    print("| `%s` | %d | %.1f | %.1f | %.1f | %s |" % (k, a[0], a[1] / 1e3, a[1] / a[0], a[2] / 1e9, sh))
# the FP16 kind's launches: single-CTA k_gemm_tc<0> and CTA-pair k_gemm_tc2<0>
# (older lists name the pair kernel without a template argument)
keys = [k for k in agg if k in ("k_gemm_tc<0>", "k_gemm_tc2<0>", "k_gemm_tc2")]
a = [sum(agg[k][0] for k in keys), sum(agg[k][1] for k in keys), sum(agg[k][2] for k in keys)]
json.dump({"kernel": "k_gemm_tc<KIND_F16> + k_gemm_tc2<KIND_F16>", "launches": a[0], "dram_bytes_total": a[2],
           "dram_bytes_per_launch": a[2] / a[0],
           "per_kernel": {k: {"launches": agg[k][0], "dram_bytes_per_launch": agg[k][2] / agg[k][0]} for k in keys},
           "source": (sys.argv[2] if len(sys.argv) > 2 else src) + ": ncu --metrics "
                     "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none of "
                     "`bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 --no-variants` "
                     "(tools/r02_final.sh)"},
          open("profiles/ncu_traffic.json", "w"), indent=1)
if len(sys.argv) > 2:
    with open(src, "rb") as f, gzip.open(sys.argv[2], "wb") as g:
        shutil.copyfileobj(f, g)

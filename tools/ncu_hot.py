"""Aggregate warp-stall samples of an ncu report per CUDA source line, with
the dominant stall reasons.  usage: python tools/ncu_hot.py report.ncu-rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, cur, agg, fname = None, None, {}, "?"
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, r[0], r[1][:90])
        continue
    try:
        s = int(r[4]); ins = int(r[7])
    except ValueError:
        continue
    e = agg.setdefault(cur, [0, 0, {}])
    e[0] += s; e[1] += ins
    for i, h in reasons:
        try:
            v = int(r[i])
        except ValueError:
            continue
        if v:
            e[2][h[6:]] = e[2].get(h[6:], 0) + v
tot = sum(v[0] for v in agg.values()) or 1
print("total stall samples", tot)
for k, (s, ins, rs) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    why = ",".join(f"{n}:{c}" for n, c in sorted(rs.items(), key=lambda x: -x[1])[:3])
    print(f"{s:7d} {100*s/tot:5.1f}% ins={ins:8d} {k[0]}:{k[1]} [{why}] {k[2][:70]}")

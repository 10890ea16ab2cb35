"""Development: predict a plan's DAG critical path on the CPU from the op
times of an earlier measured run (tools/critpath.py --json), matched by (type,
gemm class, level, rect); unmatched ops get --default-us.
    python tools/crit_predict.py MEASURED.json --n 16384 [--opt key=value] [--default-us 3]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08082_b200 as tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("measured")
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--cfg", default="[F16, F16, F16, F32]")
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--default-us", type=float, default=3.0)
ap.add_argument("--show", type=int, default=0)
args = ap.parse_args()
m = json.load(open(args.measured))
t = {}
for o in m["ops"]:
    t[(o["type"], o["gclass"], o["level"], tuple(o["rect"]))] = o["ms"]
plan = tc.Plan(args.n, args.b, args.cfg)
for kv in args.opt:
    k, v = kv.split("=")
    plan.set_option(k, int(v))
N = plan.stats()["ops"]
infos = [plan.op_info(i) for i in range(N)]
deps = [plan.op_deps(i) for i in range(N)]
ms = []
miss = 0
for inf in infos:
    k = (inf["type"], inf["gclass"], inf["level"], tuple(inf["rect"]))
    if k in t:
        ms.append(t[k])
    else:
        miss += 1
        # unmatched: fixed cost + flops at a class rate (tc16 1.2 PF/s, FP32 classes 0.12 PF/s)
        rate = 1.2e15 if inf["gclass"] == "tc16" else 1.2e14
        ms.append(args.default_us * 1e-3 + (inf["flops"] / rate * 1e3 if inf["type"] == "gemm" else 0.0))
fin = [0.0] * N
via = [-1] * N
for i in range(N):
    s, v = 0.0, -1
    for d in deps[i]:
        if fin[d] > s:
            s, v = fin[d], d
    fin[i] = s + ms[i]
    via[i] = v
end = max(range(N), key=lambda i: fin[i])
path = []
i = end
while i >= 0:
    path.append(i)
    i = via[i]
print(json.dumps({"n": args.n, "ops": N, "unmatched": miss, "critical_ms": fin[end], "critical_ops": len(path),
                  "measured_critical_ms": m["summary"]["critical_ms"]}))
for i in reversed(path[:args.show]):
    print(i, infos[i]["type"], infos[i]["gclass"], infos[i]["level"], infos[i]["rect"], "%.1f us" % (ms[i] * 1e3))

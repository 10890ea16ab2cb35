"""Development: where the C3 step's time goes in the real DAG graph.  One
graph run with a timer stamp after every op (Plan.trace); an op's interval
is [latest end of its deps, its own end].  Prints, per time bin, the GEMM
flop rate and how many leaf POTRFs finished (the chain's progress).
    python tools/trace_bins.py [--n 65536] [--bin 4] [--opt key=value]..."""
import argparse
import collections
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--bin", type=float, default=4.0)
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--json", default="")
args = ap.parse_args()
plan = tc.Plan(args.n, 256, "[F16, F16, F16, F32]")
for kv in args.opt:
    if kv.startswith("g:"):  # process-wide kernel option
        tc.set_global_option(kv[2:].split("=")[0], int(kv.split("=")[1]))
    else:
        plan.set_option(kv.split("=")[0], int(kv.split("=")[1]))
a = tc.spd_generate_device(args.n, 42)
l = torch.empty_like(a)
plan.factor_device(a, l)
torch.cuda.synchronize()
te = plan.trace(a, l)
n = len(te)
info = [plan.op_info(i) for i in range(n)]
deps = [plan.op_deps(i) for i in range(n)]
if args.json:
    import json
    json.dump({"opt": args.opt, "n": args.n, "te": te, "info": info, "deps": deps,
               "probs": [plan.op_probs(i) if info[i]["type"] == "gemm" else [] for i in range(n)]},
              open(args.json, "w"))
ts = [max([te[d] for d in deps[i]], default=0.0) for i in range(n)]
span = max(te)
nb = int(span / args.bin) + 1
fl = [0.0] * nb
npot = [0] * nb
cls = [collections.Counter() for _ in range(nb)]
for i in range(n):
    s, e = ts[i], te[i]
    k = info[i]["type"] + ("/" + info[i]["gclass"] if info[i]["gclass"] else "")
    if info[i]["type"] == "potrf":
        npot[min(nb - 1, int(e / args.bin))] += 1
    d = max(e - s, 1e-6)
    for b in range(int(s / args.bin), min(nb, int(e / args.bin) + 1)):
        ov = min(e, (b + 1) * args.bin) - max(s, b * args.bin)
        if ov > 0:
            fl[b] += info[i]["flops"] * ov / d
            cls[b][k] += ov
print(args.opt, f"n={args.n} span {span:.2f} ms (stamped graph), bins of {args.bin} ms")
print("    t_ms  GEMM_TF/s  potrf_done  ready->end ms per class")
for b in range(nb):
    top = ", ".join(f"{k} {v:.1f}" for k, v in cls[b].most_common(3))
    print(f"{b * args.bin:8.1f} {fl[b] / (args.bin * 1e-3) / 1e12:9.1f} {npot[b]:6d}   {top}")

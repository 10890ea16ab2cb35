"""Development: concurrency timeline of one factorization (eager, timing
events around every op).  Prints the span, busy time per op class, and how
long each set of concurrently running classes lasted."""
import argparse
import collections
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--cfg", default="[F16, F16, F16, F32]")
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--json", default="")
args = ap.parse_args()
plan = tc.Plan(args.n, 256, args.cfg)
for kv in args.opt:
    k, v = kv.split("=")
    plan.set_option(k, int(v))
a = tc.spd_generate_device(args.n, 42)
l = torch.empty_like(a)
plan.factor_device(a, l)
t0, t1 = plan.timeline(a, l)
n = len(t0)
info = [plan.op_info(i) for i in range(n)]
key = lambda f: f["type"] + ("/" + f["gclass"] if f["gclass"] else "")
span = max(t1) - min(t0)
busy = collections.Counter()
for i in range(n):
    busy[key(info[i])] += t1[i] - t0[i]
# sweep: intervals with the set of active classes
ev = sorted([(t0[i], 1, i) for i in range(n)] + [(t1[i], -1, i) for i in range(n)])
active = collections.Counter()
last = ev[0][0]
combo = collections.Counter()
for t, d, i in ev:
    if t > last:
        kset = tuple(sorted(k for k, c in active.items() if c > 0)) or ("idle",)
        combo[kset] += t - last
        last = t
    active[key(info[i])] += d
print(json.dumps({"n": args.n, "span_ms": span, "ops": n}))
print("busy ms per class:", {k: round(v, 2) for k, v in busy.most_common()})
print("time by set of concurrently active classes (top 25):")
for k, v in combo.most_common(25):
    print(f"  {v:8.2f} ms  {'+'.join(k)}")
if args.json:
    json.dump({"t0": t0, "t1": t1, "info": info}, open(args.json, "w"))

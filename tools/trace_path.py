"""Development: the executed critical path of a traced graph run
(tools/trace_bins.py --json): from the last op back through the dependency
that finished last.  For each op: ready time (latest dep end), end time,
wait+run = end - ready, class and shape.
    python tools/trace_path.py TRACE.json [--min-ms 0.2]"""
import argparse
import collections
import json

ap = argparse.ArgumentParser()
ap.add_argument("trace")
ap.add_argument("--min-ms", type=float, default=0.2)
args = ap.parse_args()
t = json.load(open(args.trace))
te, info, deps, probs = t["te"], t["info"], t["deps"], t["probs"]
n = len(te)
ready = [max([te[d] for d in deps[i]], default=0.0) for i in range(n)]
i = max(range(n), key=lambda k: te[k])
path = []
while True:
    path.append(i)
    if not deps[i]:
        break
    i = max(deps[i], key=lambda d: te[d])
path.reverse()
agg = collections.Counter()
cnt = collections.Counter()
for i in path:
    f = info[i]
    k = f["type"] + ("/" + f["gclass"] if f["gclass"] else "")
    agg[k] += te[i] - ready[i]
    cnt[k] += 1
print(t["opt"], "n", t["n"], "span %.2f ms, executed path %d ops" % (max(te), len(path)))
for k, v in agg.most_common():
    print("  %-14s %8.2f ms over %4d ops (%.1f us each)" % (k, v, cnt[k], 1e3 * v / cnt[k]))
print("ops on the path with end - ready >= %.2f ms:" % args.min_ms)
for i in path:
    d = te[i] - ready[i]
    if d >= args.min_ms:
        f = info[i]
        pr = probs[i]
        shape = ("%d probs %dx%dx%d%s" % (len(pr), pr[0]["m"], pr[0]["n"], pr[0]["k"], " lower" if pr[0]["lower"] else "")) if pr else str(f["rect"])
        print("  op %5d %-12s ready %8.2f end %8.2f (%6.2f ms) %s flops %.2e" %
              (i, f["type"] + "/" + (f["gclass"] or ""), ready[i], te[i], d, shape, f["flops"]))

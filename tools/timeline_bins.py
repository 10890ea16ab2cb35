"""Development: GEMM flop rate over the time of one eager multi-stream
factorization (plan.timeline events), in bins: where the step leaves the
tensor pipe idle (start-up, chain-bound stretches, tail)."""
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
args = ap.parse_args()
plan = tc.Plan(args.n, 256, "[F16, F16, F16, F32]")
for kv in args.opt:
    plan.set_option(kv.split("=")[0], int(kv.split("=")[1]))
a = tc.spd_generate_device(args.n, 42)
l = torch.empty_like(a)
plan.factor_device(a, l)
t0, t1 = plan.timeline(a, l)
n = len(t0)
info = [plan.op_info(i) for i in range(n)]
base = min(t0)
span = max(t1) - base
nb = int(span / args.bin) + 1
fl = [0.0] * nb
act = [collections.Counter() for _ in range(nb)]
for i in range(n):
    s, e = t0[i] - base, t1[i] - base
    k = info[i]["type"] + ("/" + info[i]["gclass"] if info[i]["gclass"] else "")
    d = max(e - s, 1e-6)
    for b in range(int(s / args.bin), min(nb, int(e / args.bin) + 1)):
        ov = min(e, (b + 1) * args.bin) - max(s, b * args.bin)
        if ov > 0:
            fl[b] += info[i]["flops"] * ov / d
            act[b][k] += ov
print(args.opt)
print(f"n={args.n} span {span:.2f} ms, bins of {args.bin} ms: GEMM TF/s and busy ms per class")
for b in range(nb):
    top = ", ".join(f"{k} {v:.1f}" for k, v in act[b].most_common(4))
    print(f"{b * args.bin:7.1f} {fl[b] / (args.bin * 1e-3) / 1e12:8.1f}  {top}")

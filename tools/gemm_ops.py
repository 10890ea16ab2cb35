"""Where the tcgen05 GEMM time goes at C3 (development): serialized per-op
device time of every GEMM op of one N=65536 factorization, grouped by the
op's shape class, sorted by time lost against the burst peak.

    python tools/gemm_ops.py [n] [peak_tflops]
"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("TC_ROOT", ROOT))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 1625.0
a = tc.spd_generate_device(n, 42)
l = torch.empty_like(a)
plan = tc.Plan(n, 256, "[F16, F16, F16, F32]")
plan.factor_device(a, l)
ms = plan.profile(a, l)
groups = collections.defaultdict(lambda: [0, 0.0, 0.0, 0])
rows = []
for i, t in enumerate(ms):
    info = plan.op_info(i)
    if info["type"] != "gemm":
        continue
    probs = plan.op_probs(i)
    key = (info["gclass"], len(probs), probs[0]["m"], probs[0]["n"], probs[0]["k"], probs[0]["exec_level"],
           probs[0]["lower"])
    g = groups[key]
    g[0] += 1
    g[1] += t
    g[2] += info["flops"]
    tiles = sum(((p["m"] + 127) // 128) * ((p["n"] + 255) // 256) for p in probs)
    g[3] = tiles
tot = sum(v[1] for v in groups.values())
print(f"n={n}: GEMM ops serialized {tot:.2f} ms")
print(f"{'class':6s} {'probs':>5s} {'m':>6s} {'n':>6s} {'k':>6s} ex lo {'cnt':>4s} {'tiles':>6s} {'ms':>8s} "
      f"{'TF/s':>7s} {'lost ms':>8s}")
out = []
for k, v in groups.items():
    tf = v[2] / (v[1] * 1e-3) / 1e12 if v[1] else 0
    lost = v[1] - v[2] / (peak * 1e12) * 1e3
    out.append((lost, k, v, tf))
for lost, k, v, tf in sorted(out, reverse=True)[:40]:
    print(f"{k[0]:6s} {k[1]:5d} {k[2]:6d} {k[3]:6d} {k[4]:6d} {k[5]:2d} {k[6]:2d} {v[0]:4d} {v[3]:6d} {v[1]:8.3f} "
          f"{tf:7.1f} {lost:8.3f}")

"""development: run-to-run bit determinism of one factorization; where two
runs differ (256-blocks of the lower triangle), per execution mode"""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
mode = sys.argv[2] if len(sys.argv) > 2 else "graph"
cfg = "[F16, F16, F16, F32]"
a = tc.spd_generate_device(n, 42)
plan = tc.Plan(n, 256, cfg)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    plan.set_option(k, int(v))
if mode == "eager":
    plan.set_option("use_graph", 0)
if mode == "serial":
    plan.set_option("use_graph", 0)
    plan.set_option("n_streams", 1)
outs = []
for r in range(3):
    l = a.clone()
    assert plan.factor_device(a, l).status == "ok"
    outs.append(l)
B = 256
nb = n // B
res = {"n": n, "mode": mode, "opts": sys.argv[3:]}
for k in (1, 2):
    d = (outs[0] != outs[k])
    # column-major tensor t[j, i] = A(i, j): blocks
    db = d.view(nb, B, nb, B).any(dim=3).any(dim=1)  # [jb, ib]
    idx = db.nonzero().tolist()
    res["run%d_diff_blocks" % k] = len(idx)
    res["run%d_first" % k] = [(ib, jb) for jb, ib in idx[:12]]
    if len(idx):
        res["run%d_maxabs" % k] = float((outs[0] - outs[k]).abs().max())
print(json.dumps(res))

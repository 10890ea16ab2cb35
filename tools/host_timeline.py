"""Development: timeline of the host entry point (eager): when each H2D /
D2H copy completes relative to the compute ops, to see where the end-to-end
time goes (PCIe idle gaps, D2H waiting for final blocks)."""
import argparse
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--cfg", default="[F16, F16, F16, F32]")
ap.add_argument("--json", default="")
ap.add_argument("--graph", type=int, default=1, help="1: stamped DAG graph (the real path); 0: eager with events")
args = ap.parse_args()
n = args.n
plan = tc.Plan(n, 256, args.cfg)
a = tc.spd_generate_device(n, 42)
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
host.copy_(a)
del a
torch.cuda.empty_cache()
hnp = host.numpy().T
plan.factor_host(hnp)  # warm: staging buffer, plans
n_ops = plan.stats()["ops"]
infos = [plan.op_info(i) for i in range(n_ops)]
n_exp = sum(1 for f in infos if f["type"] == "export")
n_blk = 8 * n // 256 + 4096  # >= H2D copy chunks
lib = tc.lib()
if args.graph:
    # the host entry point's own DAG graph, stamped: completion times only
    t1, th, td = (C.c_float * n_ops)(), (C.c_float * n_blk)(), (C.c_float * n_blk)()
    rc = lib.tc_plan_trace_host(plan._h, C.c_void_p(host.data_ptr()), n, None, t1, n_ops, th, n_blk, td, n_blk)
    assert rc == 0, rc
    t1 = list(t1)
    t0 = list(t1)
else:
    t0, t1 = (C.c_float * n_ops)(), (C.c_float * n_ops)()
    th, td = (C.c_float * n_blk)(), (C.c_float * n_exp)()
    rc = lib.tc_plan_timeline_host(plan._h, C.c_void_p(host.data_ptr()), n, None, t0, t1, n_ops, th, n_blk, td, n_exp)
    assert rc == 0, rc
    t0, t1 = list(t0), list(t1)
th, td = [x for x in th if x > -1e8 and x != 0], [x for x in td if x > -1e8 and x != 0]
comp = [i for i in range(n_ops) if infos[i]["type"] not in ("import", "export")]
span = max(max(t1), max(td))
print(json.dumps({"n": n, "span_ms": span, "h2d_last_ms": max(th), "d2h_first_ms": min(td), "d2h_last_ms": max(td),
                  "compute_first_ms": min(t0[i] for i in comp), "compute_last_ms": max(t1[i] for i in comp)}))
# fraction of the D2H stream by time: cumulative exported bytes vs time
rects = [infos[i] for i in range(n_ops) if infos[i]["type"] == "export"]
print("h2d completions (every 1/16):", [round(th[int(k * (len(th) - 1) / 16)], 1) for k in range(17)])
print("d2h completions (every 1/16):", [round(td[int(k * (len(td) - 1) / 16)], 1) for k in range(17)])
# compute activity in 20 ms buckets
B = 20.0
nb = int(span // B) + 1
busy = [0.0] * nb
for i in comp:
    s, e = t0[i], t1[i]
    k = int(s // B)
    while s < e and k < nb:
        hi = min(e, (k + 1) * B)
        busy[k] += hi - s
        s = hi
        k += 1
print("compute busy ms (sum over ops) per 20 ms bucket:", [round(x, 1) for x in busy])
done = [0] * nb
for i in comp:
    done[min(nb - 1, int(t1[i] // B))] += 1
print("compute ops completed per 20 ms bucket:", done)
fl = [0.0] * nb
for i in comp:
    fl[min(nb - 1, int(t1[i] // B))] += infos[i]["flops"]
print("TFLOP completed per 20 ms bucket:", [round(x / 1e12, 1) for x in fl])
import time  # noqa: E402
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t = time.perf_counter()
    plan.factor_host(hnp)
    ts.append(time.perf_counter() - t)
fl = n ** 3 / 3.0
print("factor_host wall s:", [round(x, 4) for x in ts], "-> %.1f TFLOP/s (nominal n^3/3)" % (fl / min(ts) / 1e12))
if args.json:
    json.dump({"t0": t0, "t1": t1, "h2d": th, "d2h": td, "info": infos}, open(args.json, "w"))

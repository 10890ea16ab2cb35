"""development: run-to-run variance of the C4 batch call (16 systems, 8 plans)"""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
from paper_2601_08082_b200.batch import synthetic_spd_device
n = 16384
batch = tc.Batch(n, 256, "[F16, F16, F16, F32]", True, 8)
a_list = [synthetic_spd_device(n, 1000 + k) for k in range(16)]
src = [a.clone() for a in a_list]
batch.run(a_list)
order = int(sys.argv[1]) if len(sys.argv) > 1 else 1
batch.set_option("solve_order", order)
for solve in (0, 1):
    ts = []
    for rep in range(16 if solve else 6):
        for a, s in zip(a_list, src):
            a.copy_(s)
        b_list = [a.sum(dim=0, keepdim=True).contiguous() for a in a_list] if solve else None
        torch.cuda.synchronize()
        t = time.perf_counter()
        st = batch.run(a_list, b_list) if solve else batch.run(a_list)
        torch.cuda.synchronize()
        ts.append(round((time.perf_counter() - t) * 1e3, 1))
    print(json.dumps({"order": order, "solve": solve, "ms": ts}), flush=True)

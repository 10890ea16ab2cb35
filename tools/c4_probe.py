"""development: C4 batch timing split (factorizations only vs + solves) by batch size"""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
from paper_2601_08082_b200.batch import synthetic_spd_device
n = 16384
batch = tc.Batch(n, 256, "[F16, F16, F16, F32]", True, 8)
warm = [synthetic_spd_device(n, 10 ** 6 + k) for k in range(8)]
batch.run(warm)
del warm
for cnt in (8, 16, 24, 32):
    for solve in (0, 1):
        a_list = [synthetic_spd_device(n, 1000 + k) for k in range(cnt)]
        b_list = [a.sum(dim=0, keepdim=True).contiguous() for a in a_list] if solve else None
        torch.cuda.synchronize()
        t = time.perf_counter()
        st = batch.run(a_list, b_list) if solve else batch.run(a_list)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(json.dumps({"count": cnt, "solve": solve, "ms": round(dt * 1e3, 1), "ms_per_sys": round(dt * 1e3 / cnt, 2),
                          "ok": sum(1 for x in st if x == "ok")}), flush=True)
        del a_list, b_list

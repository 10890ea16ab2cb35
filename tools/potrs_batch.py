"""development: batched POTRS time (tc_batch solve pass) vs number of systems"""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
from paper_2601_08082_b200.batch import synthetic_spd_device
n = 16384
batch = tc.Batch(n, 256, "[F16, F16, F16, F32]", True, 16)
a_all = [synthetic_spd_device(n, 100 + k) for k in range(32)]
batch.run(a_all, [a.sum(dim=0, keepdim=True).contiguous() for a in a_all])  # factor in place + warm
for cnt in (1, 4, 8, 16, 32):
    a_list = a_all[:cnt]
    # factors already in place: time solves only via a factor-free path: potrs_device per system vs batch
    bl = [a.sum(dim=0, keepdim=True).contiguous() for a in a_list]
    torch.cuda.synchronize()
    t = time.perf_counter()
    for a, b in zip(a_list, bl):
        tc.potrs_device(a, b)
    torch.cuda.synchronize()
    seq = time.perf_counter() - t
    print(json.dumps({"systems": cnt, "sequential_potrs_ms": round(seq * 1e3, 2)}), flush=True)

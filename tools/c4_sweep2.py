"""development: C4 batch throughput vs plans per GPU and tile scheduling"""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
from paper_2601_08082_b200.batch import synthetic_spd_device
n, count = 16384, 24
mats = [synthetic_spd_device(n, 1000 + k) for k in range(8)]
fl = tc.potrf_flops(n)
for tiles in (1, 0):
    for conc in (1, 2, 4, 8):
        b = tc.Batch(n, 256, "[F16, F16, F16, F32]", True, conc)
        b.set_option("bulk_tiles_per_cta", tiles)
        b.run([m.clone() for m in mats[:conc]])  # warm
        res = []
        for rep in range(2):
            work = [m.clone() for m in mats] * (count // 8)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); st = b.run(work); e1.record(); torch.cuda.synchronize()
            res.append(count * fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
            del work
        print(json.dumps({"tiles_per_cta": tiles, "concurrency": conc, "tflops": [round(x, 1) for x in res]}), flush=True)
        del b
        torch.cuda.empty_cache()

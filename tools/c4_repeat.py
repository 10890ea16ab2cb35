"""development: C4 repeated in one process (per-batch-call device ms and the
SM clock around each), to see whether the slow C4 runs are per call."""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402
from paper_2601_08082_b200.batch import spd_generate_many, synthetic_spd_device  # noqa: E402

conc = int(sys.argv[1]) if len(sys.argv) > 1 else 16
fl = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
n = 16384
batch = tc.Batch(n, 256, "[F16, F16, F16, F32]", True, conc)
warm = [synthetic_spd_device(n, 10 ** 6 + k) for k in range(conc)]
batch.run(warm, [a.sum(dim=0, keepdim=True).contiguous() for a in warm])
del warm
torch.cuda.synchronize()
a_list = spd_generate_many(n, list(range(1000, 1000 + fl)))
orig = [a.clone() for a in a_list]
flops = tc.potrf_flops(n) + 2 * n * n


def clocks(out, stop):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip()
        out.append(r)
        time.sleep(0.05)


for rep in range(reps):
    for a, o in zip(a_list, orig):
        a.copy_(o)
    b_list = [a.sum(dim=0, keepdim=True).contiguous() for a in a_list]
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=clocks, args=(samples, stop))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = batch.run(a_list, b_list)
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"conc": conc, "in_flight": fl, "rep": rep, "ms": round(ms, 1),
                      "tflops": round(fl * flops / (ms * 1e-3) / 1e12, 1), "solve_ms": round(batch.last_solve_ms(), 1),
                      "ok": sum(x == "ok" for x in st), "clk_pw_temp": samples[:: max(1, len(samples) // 4)]}), flush=True)

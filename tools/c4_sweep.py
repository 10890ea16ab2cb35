"""development: C4 batch throughput vs plans per GPU"""
import json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_08082_b200.batch import run_batch_on_rank
for conc in (2, 4, 6, 8):
    local, tot, fl = run_batch_on_rank(32, 16384, 256, "[F16, F16, F16, F32]", seed0=1000, concurrency=conc, in_flight=8)
    print(json.dumps({"concurrency": conc, "tflops": tot.systems * fl / (tot.device_ms * 1e-3) / 1e12,
                      "ms": tot.device_ms, "failed": tot.failed}), flush=True)
    torch.cuda.empty_cache()
import paper_2601_08082_b200 as tc
for dag in (1, 0):
    a = tc.spd_generate_device(16384, 1); l = torch.empty_like(a)
    p = tc.Plan(16384, 256, "[F16, F16, F16, F32]"); p.set_option("dag_graph", dag)
    t = time.time(); p.factor_device(a, l); torch.cuda.synchronize(); build = time.time() - t
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): p.factor_device(a, l, sync=False)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"dag": dag, "first_call_s": build, "ms": e0.elapsed_time(e1) / 5}), flush=True)

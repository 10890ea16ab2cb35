"""development: C4 as the bench runs it"""
import json, sys
sys.path.insert(0, ".")
from paper_2601_08082_b200.batch import run_batch_on_rank
cfgs = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [(8, 16), (4, 16), (8, 32)]
for conc, fl in cfgs:
    local, tot, flp = run_batch_on_rank(64, 16384, 256, "[F16, F16, F16, F32]", seed0=1000, concurrency=conc, in_flight=fl)
    print(json.dumps({"conc": conc, "in_flight": fl, "tflops": tot.systems * flp / (tot.device_ms * 1e-3) / 1e12,
                      "ms": tot.device_ms, "res": tot.worst_residual}), flush=True)

"""Golden outcome of BASELINE config C2 (N=8192, b=256, "[F16, F32, F64]",
seed 42) from the oracle (oracle/oracle.c, the C restatement pinned
bit-exact against the compiled reference in tests/test_cpu.py), run in this
container with all host threads.  The compiled reference itself (SURVEY
6.2) reported rel_error 1.875941e-06 for the same input; both are stored.
Writes tests/golden/c2.json.  TEST INFRASTRUCTURE ONLY."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Oracle, parse_levels  # noqa: E402

n, b, cfg, seed = 8192, 256, "[F16, F32, F64]", 42
o = Oracle()
o.set_threads(os.cpu_count() or 1)
a = o.spd_generate(n, seed)
t0 = time.time()
st, det, _, rel, fl = o.factor(a, b, parse_levels(cfg))
out = {"n": n, "b": b, "config": cfg, "seed": seed, "status": st, "rel_error": rel, "flops": list(fl.as_tuple()),
       "oracle_seconds": time.time() - t0, "threads": o.threads(),
       "reference_rel_error_survey": 1.875941e-06}
with open(os.path.join(HERE, "c2.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))

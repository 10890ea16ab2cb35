"""development: C4 (as bench.py runs it) in a fresh process and after a C3
factorization in the same process, three batches each."""
import gc
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402
from paper_2601_08082_b200.batch import run_batch_on_rank  # noqa: E402


def c4(tag):
    for r in range(3):
        _, tot, fl = run_batch_on_rank(64, 16384, 256, "[F16, F16, F16, F32]", seed0=1000, concurrency=16, in_flight=32)
        print(json.dumps({"tag": tag, "rep": r, "tflops": round(tot.systems * fl / (tot.device_ms * 1e-3) / 1e12, 1),
                          "ms": round(tot.device_ms, 1)}), flush=True)
        gc.collect()
        torch.cuda.empty_cache()


if sys.argv[1:] == ["c3"]:
    plan = tc.Plan(65536, 256, "[F16, F16, F16, F32]")
    a = tc.spd_generate_device(65536, 42)
    l = torch.empty_like(a)
    for _ in range(3):
        plan.factor_device(a, l)
    torch.cuda.synchronize()
    plan = a = l = None
    gc.collect()
    torch.cuda.empty_cache()
    c4("after_c3")
else:
    c4("fresh")

import json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_08082_b200.batch import run_batch_on_rank
for rep in range(3):
    t = time.perf_counter()
    local, tot, flp = run_batch_on_rank(64, 16384, 256, "[F16, F16, F16, F32]", seed0=1000, concurrency=8, in_flight=16)
    print(json.dumps({"rep": rep, "ms": tot.device_ms, "wall_s": time.perf_counter() - t, "mem_GB": torch.cuda.memory_allocated() / 1e9,
                      "reserved_GB": torch.cuda.memory_reserved() / 1e9}), flush=True)

"""development: C4 as the bench runs it, under plan options.
    python tools/c4_bench.py [conc,in_flight[,key=value...]] ..."""
import json, os, sys
sys.path.insert(0, ".")
from paper_2601_08082_b200.batch import run_batch_on_rank
for arg in sys.argv[1:] or ["16,32"]:
    parts = arg.split(",")
    conc, fl = int(parts[0]), int(parts[1])
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in parts[2:] if not kv.startswith("g:")}
    import paper_2601_08082_b200 as tc
    tc.set_global_option("tc_pair_min_tiles", int(os.environ.get("TC_PAIR_MIN", "512")))
    for kv in parts[2:]:
        if kv.startswith("g:"):
            tc.set_global_option(kv[2:].split("=")[0], int(kv.split("=")[1]))
    local, tot, flp = run_batch_on_rank(64, 16384, 256, "[F16, F16, F16, F32]", seed0=1000, concurrency=conc,
                                        in_flight=fl, options=opts)
    print(json.dumps({"conc": conc, "in_flight": fl, "opts": opts,
                      "tflops": tot.systems * flp / (tot.device_ms * 1e-3) / 1e12,
                      "ms": tot.device_ms, "solve_ms": tot.solve_ms, "res": tot.worst_residual}), flush=True)

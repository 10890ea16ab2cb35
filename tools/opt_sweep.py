"""Development: graph-replay time of one factorization under plan options.
    python tools/opt_sweep.py --n 65536 --set shadow_per_block=0,syrk_split_min=16384 --set ...
Each --set is one variant (comma-separated key=value); prints one JSON line per variant
(min and median over --reps graph replays)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.environ.get("TC_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--cfg", default="[F16, F16, F16, F32]")
ap.add_argument("--set", action="append", default=[])
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
a = tc.spd_generate_device(args.n, 42)
l = torch.empty_like(a)
for var in args.set or [""]:
    # "g:key=value": a process-wide kernel option (tc_set_global_option), set before the plan's tables are built
    for kv in filter(None, var.split(",")):
        if kv.startswith("g:"):
            k, v = kv[2:].split("=")
            tc.set_global_option(k, int(v))
    plan = tc.Plan(args.n, args.b, args.cfg)
    for kv in filter(None, var.split(",")):
        if kv.startswith("g:"):
            continue
        k, v = kv.split("=")
        plan.set_option(k, int(v))
    st = plan.factor_device(a, l)
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.factor_device(a, l, sync=False)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    rel = tc.factorization_error_device(a, l) if args.n <= 65536 else None
    print(json.dumps({"n": args.n, "opts": var, "status": st.status, "min_ms": times[0],
                      "med_ms": times[len(times) // 2], "tflops": tc.potrf_flops(args.n) / times[0] / 1e9,
                      "ops": plan.stats()["ops"], "rel_error": rel}), flush=True)
    del plan
    tc.set_global_option("tc_pair_min_tiles", 512)  # the library default

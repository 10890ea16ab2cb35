"""rel_error and device time of one factorization per tc_kchunk setting
(development): python tools/kchunk_factor.py N kchunk..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("TC_ROOT", ROOT))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

n = int(sys.argv[1])
a = tc.spd_generate_device(n, 42)
for kc in [int(x) for x in sys.argv[2:]]:
    tc.set_global_option("tc_kchunk", kc)
    plan = tc.Plan(n, 256, "[F16, F16, F16, F32]")
    l = torch.empty_like(a)
    plan.factor_device(a, l)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        plan.factor_device(a, l, sync=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n} kchunk={kc} ms={e0.elapsed_time(e1) / 3:.2f} rel={tc.factorization_error_device(a, l):.6e}",
          flush=True)
    del plan, l

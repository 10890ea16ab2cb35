"""development: POTRS (forward + backward substitution) time at N"""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
from paper_2601_08082_b200.batch import synthetic_spd_device
for n in (4096, 16384, 65536):
    a = synthetic_spd_device(n, 1)
    p = tc.Plan(n, 256, "[F16, F16, F16, F32]")
    a0 = a.clone()
    p.factor_device(a)
    b = a0.sum(dim=0, keepdim=True).contiguous()
    b0 = b.clone()
    tc.potrs_device(a, b)
    x = b.clone()
    res = tc.solve_residual_device(a0, x[0].contiguous(), b0[0].contiguous())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5):
        b.copy_(b0); tc.potrs_device(a, b)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byts = n * (n + 1) * 8  # L lower triangle read twice (n(n+1)/2 * 8 B each way)
    print(json.dumps({"n": n, "potrs_ms": ms, "GBs": byts / ms / 1e6, "residual": res}), flush=True)
    del a, a0, p
    torch.cuda.empty_cache()

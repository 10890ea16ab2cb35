"""development: accuracy of the three-pass TF32 path (F32 levels on tcgen05)
against the SIMT FP32 path on the same inputs, plus the 4096^3 TF32X3 GEMM time"""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
for n, cfg in ((2048, "Pure F32"), (4096, "[F16, F32]")):
    a = tc.spd_generate_device(n, 3)
    out = {"n": n, "cfg": cfg}
    for tc32 in (1, 0):
        p = tc.Plan(n, 128, cfg)
        p.set_option("use_tc32", tc32)
        l = torch.empty_like(a)
        st = p.factor_device(a, l)
        out["rel_tc32" if tc32 else "rel_simt"] = tc.factorization_error_device(a, l)
    print(json.dumps(out), flush=True)
us = tc.debug_gemm("tc32", 4096, 4096, 4096, False, 1.0, 1, iters=10)
print(json.dumps({"tc32_4096^3_us": us, "tflops": 2 * 4096 ** 3 / us / 1e6}))

"""development: per-phase cycle counts of the leaf POTRF kernel (k_potrf.cu)"""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
f = tc.lib().tc_debug_potrf_clocks
f.argtypes = [C.POINTER(C.c_longlong), C.c_int]
out = (C.c_longlong * 8)()
for n, cfg in [(16384, "[F16, F16, F16, F32]"), (4096, "Pure F16")]:
    a = tc.spd_generate_device(n, 1)
    l = torch.empty_like(a)
    p = tc.Plan(n, 256, cfg)
    p.factor_device(a, l)
    f(out, 1)
    ms = p.profile(a, l)
    f(out, 1)
    k = max(out[5], 1)
    pot = [ms[i] for i in range(len(ms)) if p.op_info(i)["type"] == "potrf"]
    print(cfg, n, "leaves", out[5], "cycles/leaf: load %.0f a %.0f b1 %.0f b2 %.0f store %.0f | event %.1f us" % (
        out[0] / k, out[1] / k, out[2] / k, out[3] / k, out[4] / k, 1e3 * sum(pot) / max(len(pot), 1)))

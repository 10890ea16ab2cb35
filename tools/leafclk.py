"""debug: per-phase cycle counts of the leaf kernels (POTRF: a, b1, b2; TRSM block 0: sums, solve)"""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
f = tc.lib().tc_debug_leaf_clocks
f.argtypes = [C.POINTER(C.c_longlong), C.c_int]
out = (C.c_longlong * 8)()
for n, cfg in [(4096, "[F16, F16, F16, F32]"), (2048, "[F16, F32, F64]")]:
    a = tc.spd_generate_device(n, 1)
    l = torch.empty_like(a)
    p = tc.Plan(n, 256, cfg)
    p.factor_device(a, l)
    f(out, 1)
    ms = p.profile(a, l)
    f(out, 1)
    cnt, tcnt = max(out[3], 1), max(out[7], 1)
    pot = [ms[i] for i in range(len(ms)) if p.op_info(i)["type"] == "potrf"]
    trs = [ms[i] for i in range(len(ms)) if p.op_info(i)["type"] == "trsm"]
    print(cfg, "potrf x%d cycles: a %.0f b1 %.0f b2 %.0f ev %.3f ms" % (out[3], out[0] / cnt, out[1] / cnt, out[2] / cnt, sum(pot) / len(pot)),
          "| trsm x%d cycles: sums %.0f solve %.0f ev %.3f ms" % (out[7], out[4] / tcnt, out[5] / tcnt, sum(trs) / max(len(trs), 1)))

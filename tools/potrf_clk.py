"""development: per-phase cycle counts of the leaf POTRF (k_potrf.cu) and
leaf inverse (k_inverse.cu, CTA 0) kernels over one serialized factorization"""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
import paper_2601_08082_b200 as tc
fp = tc.lib().tc_debug_potrf_clocks
fi = tc.lib().tc_debug_inv_clocks
for f in (fp, fi):
    f.argtypes = [C.POINTER(C.c_longlong), C.c_int]
out = (C.c_longlong * 8)()
for n, cfg in [(16384, "[F16, F16, F16, F32]"), (4096, "Pure F16")]:
    a = tc.spd_generate_device(n, 1)
    l = torch.empty_like(a)
    p = tc.Plan(n, 256, cfg)
    p.factor_device(a, l)
    fp(out, 1)
    fi(out, 1)
    ms = p.profile(a, l)
    fp(out, 1)
    k = max(out[5], 1)
    pot = [ms[i] for i in range(len(ms)) if p.op_info(i)["type"] == "potrf"]
    inv = [ms[i] for i in range(len(ms)) if p.op_info(i)["type"] == "inverse"]
    print(cfg, n, "leaves", out[5], "potrf cycles/leaf: load %.0f a %.0f b1 %.0f b2 %.0f store %.0f fused-inverse %.0f (rows %.0f) | event %.1f us" % (
        out[0] / k, out[1] / k, out[2] / k, out[3] / k, out[4] / k, out[6] / k, out[7] / k, 1e3 * sum(pot) / max(len(pot), 1)))
    fi(out, 1)
    k = max(out[6], 1)
    print(cfg, n, "inverses", out[6], "CTA0 cycles: load %.0f rcp %.0f diag %.0f prod %.0f tri %.0f store %.0f | event %.1f us"
          % (out[0] / k, out[1] / k, out[2] / k, out[3] / k, out[4] / k, out[5] / k, 1e3 * sum(inv) / max(len(inv), 1)))

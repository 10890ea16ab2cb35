"""Accuracy probe of the factorization GEMM classes (development tool).

For each case: run one problem through tc_gemm_problem_device (the engine's
launch path), sample rows x cols, and print the error against the exact
value (x87 extended) for the GPU and for the oracle's gemm_mixed (sequential
FP32 round-to-nearest, the reference's dot_update), in units of the
destination's ulp: max, RMS, mean signed (drift), where the worst is.
Also the device time of one launch (tc_debug_gemm) per kchunk setting.

    python tools/gemm_acc_probe.py [kchunk ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402
from pyoracle import Oracle  # noqa: E402
from test_gpu_kernels import _OPERAND, _dtype, _layout, _sample  # noqa: E402

CASES = [
    ("tc16", 0, True, 256, 256, 4096),
    ("tc16", 0, False, 2048, 1024, 4096),
    ("tc16", 1, True, 256, 256, 32768),
    ("tc16", 1, False, 2048, 1024, 8192),
    ("tc32", 1, False, 2048, 1024, 4096),
]


def run(o, gclass, lvl, lower, m, n, k):
    op = _OPERAND[gclass]
    pos, rows, ldw = _layout(m, n, k, lower)
    g = torch.Generator(device="cuda").manual_seed(1000 * m + 7 * n + k)
    bufs = [None, None, None]
    for lv in {op, lvl}:
        bufs[lv] = torch.zeros((rows, ldw), dtype=_dtype(lv), device="cuda")
    ob, cb = bufs[op], bufs[lvl]
    a_rows = slice(pos["a_r0"], pos["a_r0"] + m)
    b_rows = slice(pos["b_r0"], pos["b_r0"] + n)
    ob[a_rows, :k] = (torch.rand((m, k), generator=g, device="cuda", dtype=torch.float64) * 2 - 1).to(ob.dtype)
    if not lower:
        ob[b_rows, :k] = (torch.rand((n, k), generator=g, device="cuda", dtype=torch.float64) * 2 - 1).to(ob.dtype)
    c_rows = slice(pos["c_r0"], pos["c_r0"] + m)
    c_cols = slice(pos["c_c0"], pos["c_c0"] + n)
    cb[c_rows, c_cols] = (torch.rand((m, n), generator=g, device="cuda", dtype=torch.float64) * 8 - 4).to(cb.dtype)
    c0 = cb[c_rows, c_cols].clone()
    tc.gemm_problem_device(gclass, bufs[0], bufs[1], bufs[2], ldw, m, n, k, lower=lower, exec_level=lvl, **pos)
    torch.cuda.synchronize()
    c1 = cb[c_rows, c_cols]
    rng = np.random.default_rng(k)
    ri, cj = _sample(48, m, rng), _sample(48, n, rng)
    ti, tj = torch.as_tensor(ri, device="cuda"), torch.as_tensor(cj, device="cuda")
    A = ob[a_rows, :k][ti].double().cpu().numpy()
    B = ob[b_rows, :k][tj].double().cpu().numpy()
    C0 = c0[ti][:, tj].double().cpu().numpy()
    got = c1[ti][:, tj].double().cpu().numpy()
    ref = np.asfortranarray(C0.copy())
    o.gemm_mixed(ref, np.asfortranarray(A), np.asfortranarray(B), -1.0, 1.0, lvl)
    LD = np.longdouble
    exact = C0.astype(LD) - A.astype(LD) @ B.T.astype(LD)
    keep = (ri[:, None] >= cj[None, :]) if lower else np.ones_like(got, dtype=bool)
    dt = (np.float16, np.float32, np.float64)[lvl]
    ulp = np.spacing(np.abs(exact).astype(dt)).astype(LD)
    out = {}
    for name, v in (("gpu", got), ("oracle", ref)):
        e = (v.astype(LD) - exact) / ulp
        e = e[keep]
        diag = (ri[:, None] == cj[None, :])[keep]
        out[name] = (float(np.abs(e).max()), float(np.sqrt(np.mean(e * e))), float(np.mean(e)),
                     float(np.abs(e[diag]).max()) if diag.any() else 0.0)
    return out


def main():
    o = Oracle()
    kchunks = [int(x) for x in sys.argv[1:]] or [0, 1024]
    for case in CASES:
        for kc in kchunks:
            tc.set_global_option("tc_kchunk", kc)
            r = run(o, *case)
            us = tc.debug_gemm(case[0], case[3], case[4], case[5], lower=case[2], exec_level=case[1], iters=10)
            print(f"{case} kchunk={kc:5d}  {us:9.1f} us  |err| in dest ulps: "
                  + "  ".join(f"{k}: max {v[0]:8.2f} rms {v[1]:7.2f} mean {v[2]:+8.2f} diagmax {v[3]:8.2f}"
                              for k, v in r.items()), flush=True)


if __name__ == "__main__":
    main()

"""Golden outcome of BASELINE config C4's unit system (N=16384, b=256,
"[F16, F16, F16, F32]", spd_generate seeds 0 and 1) from the oracle
(oracle/oracle.c, pinned bit-exact against the compiled reference in
tests/test_cpu.py), run in this container with all host threads.

Per seed it records the status, the flop breakdown, rel_error
(factorization_error, analysis.cpp:30-62) and the solve residual
||b - A x||_2 / (||A||_F ||x||_2 + ||b||_2) of or_potrs (the POTRS
restatement: forward sweep = trsm_leaf at Double on b^T, kernels.cpp:71-92)
for b = A * ones, computed here in numpy float64 over the full symmetric A.
tests/test_batch.py::test_c4_unit_matches_golden drives tc_batch_run on the
same inputs and asserts rel_error and residual within 2x of these.

Writes tests/golden/c4.json.  TEST INFRASTRUCTURE ONLY.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Oracle, parse_levels  # noqa: E402

N, B, CFG, SEEDS = 16384, 256, "[F16, F16, F16, F32]", (0, 1)


def rhs_of(a):
    """b = A * ones, summed in numpy (the GPU test recomputes it the same way)"""
    return a.sum(axis=1)


def residual(a, x, b):
    r = b - a @ x
    return float(np.linalg.norm(r) / (np.linalg.norm(a) * np.linalg.norm(x) + np.linalg.norm(b)))


def main():
    o = Oracle()
    o.set_threads(os.cpu_count() or 1)
    out = {"n": N, "b": B, "config": CFG, "rhs": "b = A * ones (numpy a.sum(axis=1))",
           "residual": "||b - A x||_2 / (||A||_F ||x||_2 + ||b||_2)", "threads": o.threads(), "cases": []}
    for seed in SEEDS:
        a = o.spd_generate(N, seed)
        t0 = time.time()
        st, det, l, rel, fl = o.factor(a, B, parse_levels(CFG))
        t1 = time.time()
        b = rhs_of(a)
        x = o.potrs(l, b)[:, 0]
        res = residual(a, x, b)
        case = {"seed": seed, "status": st, "detail": det, "rel_error": rel, "flops": list(fl.as_tuple()),
                "potrs_residual": res, "oracle_seconds": t1 - t0}
        out["cases"].append(case)
        print(json.dumps(case), flush=True)
        del a, l
    with open(os.path.join(HERE, "c4.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

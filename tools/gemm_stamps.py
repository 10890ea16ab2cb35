"""Development: per-launch device time of k_gemm_tc at small / mid shapes and
CTA 0's phase stamps (ns from kernel entry), to see where a short launch's
fixed cost goes.  python tools/gemm_stamps.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08082_b200 as tc  # noqa: E402

names = ["setup", "tma0", "stage0", "acc", "epi_done", "exit", "c_staged", "epi_math", "epi_sync", "stores",
         "epi_end", "tld0_in", "tld0_out", "math0"]
for cls, m, n, k, lower, beta, ex in [("tc16", 128, 256, 64, 0, 1.0, 0), ("tc16", 128, 256, 512, 0, 1.0, 0),
                                      ("tc16", 2048, 256, 512, 0, 0.0, 0), ("tc16", 8192, 256, 512, 0, 0.0, 0),
                                      ("tc16", 32768, 256, 512, 0, 0.0, 0), ("tc16", 32768, 256, 256, 0, 1.0, 0),
                                      ("tc16", 8192, 1024, 1024, 0, 1.0, 0), ("tc16", 4096, 4096, 4096, 0, 1.0, 0),
                                      ("tc32", 256, 256, 256, 1, 1.0, 1), ("tc32", 4096, 256, 256, 0, 0.0, 1),
                                      ("tc32", 4096, 2048, 2048, 0, 1.0, 1), ("mma32w", 256, 256, 256, 0, 0.0, 1),
                                      ("mma32w", 4096, 256, 256, 0, 0.0, 1), ("mma32", 256, 256, 256, 1, 1.0, 1)]:
    us = tc.debug_gemm(cls, m, n, k, lower=bool(lower), beta=beta, exec_level=ex, iters=50)
    st = tc.debug_gemm_stamps() if cls.startswith("tc") else []
    fl = (m * n * k if lower else 2 * m * n * k)
    print(json.dumps({"class": cls, "m": m, "n": n, "k": k, "lower": lower, "us": round(us, 2),
                      "tflops": round(fl / us / 1e6, 1),
                      "stamps_us": {nm: (round(v / 1e3, 2) if v is not None else None) for nm, v in zip(names, st)}}))

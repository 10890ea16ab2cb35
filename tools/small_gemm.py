"""Per-launch device time of the small GEMMs on the factorization chain
(development): tc_debug_gemm = back-to-back launches in a CUDA graph.
    python tools/small_gemm.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("TC_ROOT", ROOT))
import paper_2601_08082_b200 as tc  # noqa: E402

CASES = [("tc16", 2048, 256, 512, 0, 0), ("tc16", 32768, 256, 512, 0, 0), ("tc16", 8192, 256, 256, 0, 0),
         ("tc32", 512, 256, 256, 0, 1), ("tc32", 4096, 256, 256, 0, 1), ("tc32", 256, 256, 512, 1, 1),
         ("tc32", 256, 256, 4096, 1, 1), ("mma32w", 256, 256, 256, 0, 1), ("mma32w", 4096, 256, 256, 0, 1),
         ("mma32", 256, 256, 256, 1, 1), ("tc16", 256, 256, 32768, 1, 1)]
for g, m, n, k, lo, ex in CASES:
    us = tc.debug_gemm(g, m, n, k, lower=bool(lo), exec_level=ex, iters=50)
    print(f"{g:7s} {m:6d} x {n:4d} x {k:6d} lower={lo} exec={ex}: {us:8.2f} us  "
          f"{2 * m * n * k / (us * 1e-6) / 1e12 / (2 if lo else 1):8.1f} TF/s", flush=True)

"""fixed per-launch cost of the tensor-core GEMM (development): one tile,
growing k; many tiles, k = 64 -- tc_debug_gemm back-to-back graph launches"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_08082_b200 as tc  # noqa: E402

for g, ex in (("tc16", 0), ("tc16", 1), ("tc32", 1), ("mma32", 1), ("mma32w", 1)):
    for m, n, k in ((128, 256, 64), (128, 256, 512), (128, 256, 4096), (2048, 256, 64), (16384, 256, 64),
                    (2048, 256, 512)):
        if g.startswith("mma32") and m > 4096:
            continue
        us = tc.debug_gemm(g, m, n, k, exec_level=ex, iters=50)
        print(f"{g:7s} exec={ex} {m:6d} x {n:4d} x {k:5d}: {us:8.2f} us", flush=True)

"""fixed per-launch cost split (development): beta = 0 (C never read) vs 1"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_08082_b200 as tc  # noqa: E402

for g, ex in (("tc16", 0), ("tc16", 1), ("tc32", 1)):
    for beta in (0.0, 1.0):
        for m, n, k in ((128, 256, 64), (128, 256, 512), (2048, 256, 512)):
            us = tc.debug_gemm(g, m, n, k, beta=beta, exec_level=ex, iters=50)
            print(f"{g:5s} exec={ex} beta={beta} {m:6d} x {n:4d} x {k:5d}: {us:8.2f} us", flush=True)
print("stamps (ns from entry: setup, TMA issued, stage landed, acc ready, epilogue done, exit)")
for g, ex in (("tc16", 0), ("tc16", 1), ("tc32", 1)):
    for m, n, k in ((128, 256, 64), (128, 256, 512)):
        us = tc.debug_gemm(g, m, n, k, exec_level=ex, iters=20)
        print(f"{g:5s} exec={ex} {m} x {n} x {k}: {us:7.2f} us  {tc.debug_gemm_stamps()}", flush=True)

"""one launch of a GEMM class (for single-kernel ncu captures):
    python tools/one_gemm.py gclass m n k lower exec"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_08082_b200 as tc  # noqa: E402

g, m, n, k, lo, ex = sys.argv[1], *map(int, sys.argv[2:7])
print(tc.debug_gemm(g, m, n, k, lower=bool(lo), exec_level=ex, iters=1))

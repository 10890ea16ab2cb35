"""development: fixed per-launch cost of the grouped GEMM kernels"""
import json, sys
sys.path.insert(0, ".")
import paper_2601_08082_b200 as tc
for cls in ("tc16", "tc32", "mma32"):
    for (m, n, k, beta) in [(128, 128, 64, 0.0), (128, 128, 64, 1.0), (128, 256, 256, 0.0), (256, 256, 256, 0.0),
                            (1024, 256, 256, 0.0), (4096, 256, 256, 0.0), (4096, 256, 256, 1.0), (16384, 256, 256, 0.0)]:
        ex = 0 if cls == "tc16" else 1
        us = tc.debug_gemm(cls, m, n, k, False, beta, ex, iters=50)
        print(json.dumps({"cls": cls, "m": m, "n": n, "k": k, "beta": beta, "us": round(us, 2)}), flush=True)

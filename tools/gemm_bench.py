"""Development: time single grouped-GEMM launches (tools for kernel tuning)."""
import json
import sys

sys.path.insert(0, __import__("os").environ.get("TC_ROOT", "."))
import paper_2601_08082_b200 as tc  # noqa: E402

SHAPES = [  # (m, n, k, lower, beta, exec)
    (8192, 256, 512, 0, 0.0, 0), (8192, 256, 256, 0, 1.0, 0), (32768, 256, 512, 0, 0.0, 0),
    (32768, 256, 256, 0, 1.0, 0), (4096, 4096, 4096, 0, 1.0, 0), (8192, 8192, 8192, 0, 1.0, 0),
    (16384, 16384, 16384, 0, 1.0, 0), (256, 256, 4096, 1, 1.0, 1), (2048, 2048, 4096, 0, 1.0, 1),
]
for cls in sys.argv[1:] or ["tc16", "tc32", "simt_f32"]:
    for (m, n, k, lo, beta, ex) in SHAPES:
        if cls != "tc16" and ex == 0:
            ex = 2 if cls == "simt_f64" else 1
        if cls == "simt_f64":
            ex = 2
        if cls != "tc16" and m * n * k > 2 ** 36:
            continue
        us = tc.debug_gemm(cls, m, n, k, bool(lo), beta, ex, iters=10)
        fl = (m * n * k if lo else 2 * m * n * k)
        print(json.dumps({"cls": cls, "m": m, "n": n, "k": k, "lower": lo, "beta": beta, "us": round(us, 2),
                          "tflops": round(fl / us / 1e6, 1)}), flush=True)

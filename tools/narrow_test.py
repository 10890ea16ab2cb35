"""development: the narrow FP16 kind (KIND_F16N, 128x128 tiles) against the
128x256 kind on the same inputs (bit-for-bit), then per-launch times of both
on the skinny shapes of the TRSM recursion."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("TC_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

tc.set_global_option("tc_pair_min_tiles", 0)


def run(narrow, m, n, k, ex, lower, beta, seed=0):
    tc.set_global_option("tc_narrow_max_tiles", 1 << 30 if narrow else 0)
    g = torch.Generator(device="cuda").manual_seed(seed)
    R = max(m + n, m + 1)
    ldw = ((k + n + 63) // 64) * 64
    b16 = (torch.rand((R, ldw), device="cuda", generator=g) * 2 - 1).half()
    b32 = torch.rand((R, ldw), device="cuda", generator=g) * 2 - 1
    b_r0 = 0 if lower else m
    tc.gemm_problem_device("tc16", b16, b32, None, ldw, m, n, k, 0, 0, b_r0, 0, 0, k, ex, lower, -1.0, beta)
    torch.cuda.synchronize()
    return (b16 if ex == 0 else b32)[:m, k:k + n].clone()


ok = True
for m, n, k, ex, lower, beta in [(512, 512, 512, 0, 0, 1.0), (1024, 768, 1024, 1, 0, 1.0), (300, 200, 333, 0, 0, 1.0),
                                 (512, 512, 2048, 1, 1, 1.0), (2304, 1280, 640, 1, 0, 1.0), (8192, 256, 512, 1, 0, 1.0),
                                 (256, 256, 4096, 1, 1, 1.0), (1000, 136, 200, 0, 0, 0.0)]:
    a = run(False, m, n, k, ex, lower, beta)
    b = run(True, m, n, k, ex, lower, beta)
    same = torch.equal(a.view(torch.int16) if ex == 0 else a.view(torch.int32),
                       b.view(torch.int16) if ex == 0 else b.view(torch.int32))
    ok &= same
    print(json.dumps({"m": m, "n": n, "k": k, "ex": ex, "lower": lower, "bit_identical": same,
                      "maxdiff": (a.float() - b.float()).abs().max().item()}), flush=True)
for ex in (1, 0):
    for m, n, k in [(2048, 256, 512), (4096, 256, 512), (8192, 256, 512), (16384, 256, 512), (32768, 256, 512),
                    (8192, 256, 256), (32768, 256, 256), (8192, 512, 512), (16384, 512, 512), (8192, 1024, 1024),
                    (4096, 2048, 2048)]:
        tc.set_global_option("tc_narrow_max_tiles", 0)
        t1 = tc.debug_gemm("tc16", m, n, k, exec_level=ex, iters=20)
        tc.set_global_option("tc_narrow_max_tiles", 1 << 30)
        t2 = tc.debug_gemm("tc16", m, n, k, exec_level=ex, iters=20)
        tc.set_global_option("tc_narrow_max_tiles", 0)
        print(json.dumps({"ex": ex, "m": m, "n": n, "k": k, "tiles256": (m // 128) * ((n + 255) // 256),
                          "us_wide": round(t1, 2), "us_narrow": round(t2, 2)}), flush=True)
print("ALL_BIT_IDENTICAL" if ok else "DIFFERENT")

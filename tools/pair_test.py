"""development: the CTA-pair GEMM (k_gemm_tc2) against the single-CTA kernel
on the same inputs (bit-for-bit), then per-launch times of both."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("TC_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402


def run(pair, m, n, k, ex, lower, beta, seed=0, cls="tc16"):
    tc.set_global_option("tc_pair_min_tiles", 1 if pair else 0)
    g = torch.Generator(device="cuda").manual_seed(seed)
    R = max(m + n, m + 1)
    ldw = ((k + n + 63) // 64) * 64
    b16 = (torch.rand((R, ldw), device="cuda", generator=g) * 2 - 1).half()
    b32 = torch.rand((R, ldw), device="cuda", generator=g) * 2 - 1
    b_r0 = 0 if lower else m
    tc.gemm_problem_device(cls, b16, b32, None, ldw, m, n, k, 0, 0, b_r0, 0, 0, k, ex, lower, -1.0, beta)
    torch.cuda.synchronize()
    out = (b16 if ex == 0 else b32)[:m, k:k + n].clone()
    return out


ok = True
for m, n, k, ex, lower, beta in [(512, 512, 512, 0, 0, 1.0), (1024, 768, 1024, 1, 0, 1.0), (300, 200, 333, 0, 0, 1.0),
                                 (512, 512, 2048, 1, 1, 1.0), (4096, 4096, 4096, 0, 0, 0.0), (2304, 1280, 640, 1, 0, 1.0),
                                 (256, 256, 32768, 1, 1, 1.0)]:
    a = run(False, m, n, k, ex, lower, beta)
    b = run(True, m, n, k, ex, lower, beta)
    same = torch.equal(a.view(torch.int16) if ex == 0 else a.view(torch.int32),
                       b.view(torch.int16) if ex == 0 else b.view(torch.int32))
    diff = (a.float() - b.float()).abs().max().item()
    ok &= same
    print(json.dumps({"m": m, "n": n, "k": k, "ex": ex, "lower": lower, "bit_identical": same, "maxdiff": diff}), flush=True)
for m, n, k, lower in [(512, 512, 512, 0), (1024, 768, 1024, 0), (300, 200, 333, 0), (512, 512, 2048, 1),
                       (4096, 2048, 2048, 0), (4096, 256, 256, 0)]:
    a = run(False, m, n, k, 1, lower, 1.0, cls="tc32")
    b = run(True, m, n, k, 1, lower, 1.0, cls="tc32")
    same = torch.equal(a.view(torch.int32), b.view(torch.int32))
    ok &= same
    print(json.dumps({"tc32": 1, "m": m, "n": n, "k": k, "lower": lower, "bit_identical": same,
                      "maxdiff": (a - b).abs().max().item()}), flush=True)
for m, n, k in [(4096, 4096, 4096), (4096, 2048, 2048), (8192, 8192, 8192)]:
    t1 = tc.debug_gemm("tc32", m, n, k, exec_level=1, iters=5)
    tc.set_global_option("tc_pair_min_tiles", 1)
    t2 = tc.debug_gemm("tc32", m, n, k, exec_level=1, iters=5)
    tc.set_global_option("tc_pair_min_tiles", 0)
    print(json.dumps({"tc32": 1, "m": m, "n": n, "k": k, "us_single": t1, "us_pair": t2,
                      "tf_single": 2 * m * n * k / t1 / 1e6, "tf_pair": 2 * m * n * k / t2 / 1e6}), flush=True)
for m, n, k in [(16384, 16384, 16384), (8192, 8192, 8192), (32768, 8192, 8192), (4096, 4096, 4096), (8192, 1024, 1024)]:
    tc.set_global_option("tc_pair_min_tiles", 0)
    t1 = tc.debug_gemm("tc16", m, n, k, iters=5)
    tc.set_global_option("tc_pair_min_tiles", 1)
    t2 = tc.debug_gemm("tc16", m, n, k, iters=5)
    tc.set_global_option("tc_pair_min_tiles", 0)
    print(json.dumps({"m": m, "n": n, "k": k, "us_single": t1, "us_pair": t2, "tf_single": 2 * m * n * k / t1 / 1e6,
                      "tf_pair": 2 * m * n * k / t2 / 1e6}), flush=True)
print("ALL_BIT_IDENTICAL" if ok else "DIFFERENT")

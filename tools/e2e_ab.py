"""development: e2e (tc_potrf_host, pinned host doubles) at N=65536 with and
without per-export D2H events; the host result is compared bitwise with the
device path's L."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cfg = "[F16, F16, F16, F32]"
a = tc.spd_generate_device(n, 42)
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
hnp = host.numpy().T
ref = torch.empty_like(a)
p0 = tc.Plan(n, 256, cfg)
p0.factor_device(a, ref)
torch.cuda.synchronize()
del p0
for ee in (0, 1, 0, 1):
    plan = tc.Plan(n, 256, cfg)
    plan.set_option("export_events", ee)
    host.copy_(a)
    plan.factor_host(hnp)  # warm
    ts = []
    for _ in range(2):
        host.copy_(a)
        t0 = time.perf_counter()
        st = plan.factor_host(hnp)
        ts.append(time.perf_counter() - t0)
    # column strips: the host result against the device path's L
    same = True
    for j0 in range(0, n, 4096):
        hs = host[j0:j0 + 4096].cuda()  # rows of `host` = columns of the column-major matrix
        same &= torch.equal(torch.triu(hs, diagonal=j0), torch.triu(ref[j0:j0 + 4096], diagonal=j0))
        del hs
    print(json.dumps({"n": n, "export_events": ee, "status": st.status, "s": [round(t, 4) for t in ts],
                      "tflops": round(tc.potrf_flops(n) / min(ts) / 1e12, 1), "same_as_device": same}), flush=True)
    del plan
    torch.cuda.empty_cache()

"""development: pinned-host PCIe bandwidth on this box: H2D alone, D2H
alone, and both directions at once (two streams), 4 GB each way."""
import json
import torch

nb = 4 << 30
h1 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


for _ in range(2):
    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"h2d_gbs": round(nb / t1 / 1e9, 1), "d2h_gbs": round(nb / t2 / 1e9, 1),
                      "both_gbs_each": round(nb / t3 / 1e9, 1), "both_gbs_combined": round(2 * nb / t3 / 1e9, 1)}))

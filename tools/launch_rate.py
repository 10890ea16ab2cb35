"""Is the C4 batch launch-rate bound? (development)
1. empty-kernel launch throughput: CUDA graphs of 1000 tiny kernels replayed
   on S streams at once
2. factor-only C4 throughput vs concurrency (plans side by side)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

x = torch.zeros(1, device="cuda")
for S in (1, 4, 16):
    streams = [torch.cuda.Stream() for _ in range(S)]
    graphs = []
    for s in streams:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            x.add_(0)
            with torch.cuda.graph(g, stream=s):
                for _ in range(1000):
                    x.add_(0)
        graphs.append(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for rep in range(3):
        for s, g in zip(streams, graphs):
            with torch.cuda.stream(s):
                g.replay()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"streams": S, "launches": 3000 * S, "ms": ms, "us_per_launch": ms * 1e3 / (3000 * S)}),
          flush=True)

n = 16384
from paper_2601_08082_b200.batch import synthetic_spd_device  # noqa: E402
mats = [synthetic_spd_device(n, 1000 + k) for k in range(16)]
fl = tc.potrf_flops(n)
p = tc.Plan(n, 256, "[F16, F16, F16, F32]")
print(json.dumps({"ops": p.stats()}), flush=True)
for conc in (4, 8, 16, 32):
    b = tc.Batch(n, 256, "[F16, F16, F16, F32]", True, conc)
    work = [m.clone() for m in mats] * 2
    b.run(work[:conc])
    work = [m.clone() for m in mats] * 2
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.run(work)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"concurrency": conc, "systems": len(work), "ms": ms, "tflops": len(work) * fl / ms / 1e9}),
          flush=True)
    del b, work
    torch.cuda.empty_cache()

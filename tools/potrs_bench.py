"""POTRS bandwidth (development): single-system solves at several N and the
batched solve of C4-size systems, as algorithmic GB/s (L read once per sweep:
n(n+1) * 8 bytes per system and RHS).

    python tools/potrs_bench.py [nsys]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("TC_ROOT", ROOT))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402
from paper_2601_08082_b200.batch import synthetic_spd_device  # noqa: E402


def timed(fn, reps=5):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for poll in [int(x) for x in os.environ.get("POLL", "0").split(",")]:
  tc.set_global_option("potrs_poll", poll)
  print("poll", poll, flush=True)
  for n in (4096, 16384, 65536):
      a = synthetic_spd_device(n, 1)
      a0 = a.clone()
      tc.Plan(n, 256, "[F16, F16, F16, F32]").factor_device(a)
      b0 = a0.sum(dim=0, keepdim=True).contiguous()
      b = b0.clone()
      ms = timed(lambda: (b.copy_(b0), tc.potrs_device(a, b)))
      res = tc.solve_residual_device(a0, b[0].contiguous(), b0[0].contiguous())
      print(json.dumps({"n": n, "systems": 1, "potrs_ms": ms, "GBs": n * (n + 1) * 8 / ms / 1e6, "residual": res}),
            flush=True)
      del a, a0
      torch.cuda.empty_cache()

nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = 16384
ls = [synthetic_spd_device(n, 100 + k) for k in range(nsys)]
# a factor-shaped operand: any lower triangle with a safe diagonal (timing only)
b0 = [x.sum(dim=0, keepdim=True).contiguous() for x in ls]
bs = [x.clone() for x in b0]


def run():
    for x, y in zip(bs, b0):
        x.copy_(y)
    tc.potrs_batch_device(ls, bs)


for poll in [int(x) for x in os.environ.get("POLL", "0").split(",")]:
    tc.set_global_option("potrs_poll", poll)
    ms = timed(run, 3)
    print(json.dumps({"poll": poll, "n": n, "systems": nsys, "potrs_ms": ms, "GBs": nsys * n * (n + 1) * 8 / ms / 1e6}), flush=True)

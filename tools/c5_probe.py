"""development: the distributed driver on one GPU (world 1) at N"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402
from paper_2601_08082_b200.distributed import potrf_top_split, synthetic_pieces  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or (16384, 65536):
    a11, a21, a22, l22 = synthetic_pieces(n, 256, 42, 1, 0)
    cache = {}
    ts = []
    for it in range(3):
        res = potrf_top_split(n, 256, "[F16, F16, F16, F32]", a11=a11.clone(), a21_rows=a21.clone(),
                              a22_rows=a22.clone(), l22=l22, cache=cache)
        ts.append(res.device_ms)
    mem = torch.cuda.max_memory_allocated() / 1e9
    print(json.dumps({"n": n, "status": res.status, "ms": ts, "max_torch_alloc_gb": mem,
                      "tflops": tc.potrf_flops(n) / (min(ts[1:]) * 1e-3) / 1e12}), flush=True)
    del a11, a21, a22, l22, cache, res
    torch.cuda.empty_cache()

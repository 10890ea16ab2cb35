"""development: run the compact SYRK piece of every rank of a world alone
(python tools/syrk_ext_probe.py n b world)"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402
from paper_2601_08082_b200.distributed import syrk_partition  # noqa: E402

n, b, world = (int(x) for x in sys.argv[1:4])
n1, n2 = n // 2, n - n // 2
cfg = "[F16, F16, F16, F32]"
for r, (lo, hi) in enumerate(syrk_partition(n2, b, world)):
    ps = tc.Plan.panel_syrk_rows_ext(n2, n1, b, cfg, lo, hi)
    buf, s_lo = ps.level_buffer(0)
    print(r, (lo, hi), "rows", ps.rows, "row0", ps.row0, "window", s_lo, s_lo + buf.shape[0], "ld", buf.shape[1],
          "bytes", ps.device_bytes(), flush=True)
    buf.zero_()
    a = torch.rand((n2, hi - lo), dtype=torch.float64, device="cuda")
    st = ps.factor_device(a)
    torch.cuda.synchronize()
    print("  ", st.status, flush=True)

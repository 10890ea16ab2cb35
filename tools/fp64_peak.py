"""FP64 peaks of this B200 (development): DMMA (mma.sync m8n8k4 f64, the FP64
tensor pipe) and DFMA (SIMT) over the whole GPU; the denominators of the
Pure F64 / F64-leaf rooflines.  usage: python tools/fp64_peak.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_08082_b200 as tc  # noqa: E402

lib = tc.lib()
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = {"sms": sms}
for name, kind in (("dmma", 0), ("dfma", 1)):
    best = 0.0
    for per_sm in (1, 2, 4, 8):
        for _ in range(3):
            best = max(best, lib.tc_debug_fp64_probe(kind, 20000, sms * per_sm))
    out[name + "_tflops"] = best / 1e12
out["mma_sync_tf32_sm_tflops"] = 2 * lib.tc_debug_mma_probe(0, 20000) / 1e12
out["mma_sync_f16_sm_tflops"] = 2 * lib.tc_debug_mma_probe(1, 20000) / 1e12
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)

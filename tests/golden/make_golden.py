"""Generate tests/golden/golden.json from the COMPILED REFERENCE (oracle/_ref,
built from /root/reference/proj sources by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixture pins the oracle restatement on machines without the reference
(e.g. the GPU box): status, detail text, rel_error bits, flop breakdown, and
a SHA-256 of the factor's bytes for each case; plus the published numbers of
proj/test_output.txt that the reference reproduces.
"""
import hashlib
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import numpy as np  # noqa: E402

from pyoracle import Reference, parse_levels  # noqa: E402

CASES = [
    # n, b, config, quantize, seed, scale
    (8, 2, "Pure F64", 1, 1, 1.0),
    (7, 2, "[F16, F32]", 1, 3, 1.0),
    (64, 8, "[F16, F32]", 1, 7, 1.0),
    (96, 16, "[F16, F32]", 1, 11, 1.0),
    (128, 16, "Pure F16", 1, 2, 1.0),
    (100, 7, "[F16, F16, F16, F32]", 1, 5, 1.0),
    (200, 32, "[F16, F32, F64]", 1, 4, 1.0),
    (200, 32, "[F16, F32, F64]", 0, 4, 1.0),
    (384, 48, "[F16, F16, F32]", 1, 21, 1.0),
    (256, 32, "Pure F32", 1, 9, 1.0),
    (1024, 128, "[F16, F64]", 1, 42, 1.0),        # BASELINE config C1
    (256, 32, "[F16, F32]", 1, 4, 3.0 * 65504.0 / 0.5),  # criterion 4, quantize on
    (256, 32, "[F16, F32]", 0, 4, 3.0 * 65504.0 / 0.5),  # criterion 4, quantize off
    (512, 256, "[F16, F32]", 1, 3, 1e10),          # singular diagonal through F16 TRSM
]


def f64bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def main():
    r = Reference()
    out = {"source": "oracle/_ref (compiled /root/reference/proj sources)", "cases": []}
    for n, b, cfg, q, seed, scale in CASES:
        a = r.spd_generate(n, seed)
        if scale != 1.0:
            a = np.asfortranarray(a * scale)
        l = a.copy(order="F")
        st, det, fl = r.tree_potrf(l, b, parse_levels(cfg), q)
        rel = r.factorization_error(a, l) if st == "ok" else float("nan")
        out["cases"].append({
            "n": n, "b": b, "config": cfg, "quantize": q, "seed": seed, "scale": scale,
            "status": st, "detail": det, "rel_error": rel, "rel_error_bits": f64bits(rel) if st == "ok" else None,
            "flops": list(fl.as_tuple()), "l_sha256": hashlib.sha256(l.tobytes(order="F")).hexdigest(),
            "a_sha256": hashlib.sha256(a.tobytes(order="F")).hexdigest()})
    # static flop breakdowns at the BASELINE sizes
    out["flop_breakdown"] = []
    for n, b, cfg in [(1024, 128, "[F16, F64]"), (8192, 256, "[F16, F32, F64]"),
                      (65536, 256, "[F16, F16, F16, F32]"), (65536, 256, "Pure F16"), (65536, 256, "Pure F64"),
                      (16384, 256, "[F16, F16, F16, F32]"), (131072, 256, "[F16, F16, F16, F32]"),
                      (65536, 256, "[F16, F32, F64]")]:
        out["flop_breakdown"].append({"n": n, "b": b, "config": cfg,
                                      "flops": list(r.flop_breakdown(n, b, parse_levels(cfg)).as_tuple())})
    # half rounding known answers (test_precision.cpp:75-94)
    vals = [1.0, 65504.0, 65519.0, 65520.0, -65520.0, 1e5, 2.0 ** -25, float.fromhex("0x1.0000001p-25"),
            2.0 ** -24, -0.0, -1e-30, 3.14159, 1e-7, 2049.0, 2051.0]
    out["round_half"] = [[v, r.round_to(v, 0)] for v in vals]
    # published numbers the reference reproduces (proj/test_output.txt:17-47)
    out["published"] = {"ladder_median_digits_n1024_b64": {
        "Pure F64": 14.845, "Pure F32": 7.027, "Pure F16": 3.329, "[F16, F32]": 5.294,
        "[F16, F32, F64]": 5.294, "[F16, F16, F16, F32]": 5.181},
        "deep_vs_pure_f16_ratio": 71.0708, "offdiag_share_65536": 99.9985,
        "c1_seed42_rel_error_survey_probe": 4.871e-06}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out["cases"]), "cases")


if __name__ == "__main__":
    main()

"""CPU suite (no GPU): the oracle pinned to the reference, the host planner's
bit-exact partition and flop accounting, the config grammar, and the C ABI
library surface.  Mirrors proj/tests/test_{precision,tree,analysis}.cpp and
the acceptance criteria that need no factorization on the device."""
import hashlib
import json
import math
import os
import re
import struct

import numpy as np
import pytest

from pyoracle import Oracle, parse_levels

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


# ------------------------------------------------------------ oracle pinning
@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: f"{c['n']}-{c['b']}-{c['config']}-q{c['quantize']}")
def test_oracle_matches_golden_reference_outputs(oracle, case):
    """the C restatement reproduces the compiled reference bit for bit"""
    a = oracle.spd_generate(case["n"], case["seed"])
    if case["scale"] != 1.0:
        a = np.asfortranarray(a * case["scale"])
    assert hashlib.sha256(a.tobytes(order="F")).hexdigest() == case["a_sha256"]
    l = a.copy(order="F")
    st, det, fl = oracle.tree_potrf(l, case["b"], parse_levels(case["config"]), case["quantize"])
    assert st == case["status"]
    assert det == case["detail"]
    assert list(fl.as_tuple()) == case["flops"]
    assert hashlib.sha256(l.tobytes(order="F")).hexdigest() == case["l_sha256"]
    if st == "ok":
        assert bits(oracle.factorization_error(a, l)) == case["rel_error_bits"]


def test_oracle_round_half_golden(oracle):
    for v, want in GOLDEN["round_half"]:
        got = oracle.round_to(v, 0)
        assert (got == want and math.copysign(1, got) == math.copysign(1, want)) or (math.isnan(got) and math.isnan(want))


def test_oracle_half_rounding_exhaustive(oracle):
    """every finite binary16 value survives, midpoints tie to even
    (test_precision.cpp:22-66, 111-123), overflow at 65520"""
    h = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    for v in h[::97]:
        assert oracle.round_to(v, 0) == v
        assert oracle.round_to(-v, 0) == -v
    mids = (h[1:-1:53] + h[2::53][: len(h[1:-1:53])]) / 2
    for m in mids[:300]:
        r = oracle.round_to(m, 0)
        assert r == float(np.float16(m))  # numpy float16 is RNE
    assert oracle.round_to(65519.0, 0) == 65504.0
    assert oracle.round_to(65520.0, 0) == math.inf


def test_oracle_bit_exact_vs_compiled_reference(oracle, ref):
    """random shapes and configs, the compiled reference side by side"""
    rng = np.random.default_rng(5)
    cfgs = ["Pure F64", "Pure F32", "Pure F16", "[F16, F32]", "[F16, F32, F64]", "[F16, F16, F16, F32]"]
    for it in range(12):
        n = int(rng.integers(1, 200))
        b = int(rng.integers(1, n + 1))
        cfg = cfgs[it % len(cfgs)]
        q = bool(it % 3)
        seed = int(rng.integers(0, 1000))
        a = ref.spd_generate(n, seed)
        l1, l2 = a.copy(order="F"), a.copy(order="F")
        s1 = oracle.tree_potrf(l1, b, parse_levels(cfg), q)
        s2 = ref.tree_potrf(l2, b, parse_levels(cfg), q)
        assert s1[:2] == s2[:2]
        assert s1[2].as_tuple() == s2[2].as_tuple()
        assert np.array_equal(l1.view(np.uint64), l2.view(np.uint64))


def test_oracle_kernels_vs_reference(oracle, ref):
    rng = np.random.default_rng(9)
    for level in (0, 1, 2):
        m, n, k = 7, 5, 9
        a = np.asfortranarray(rng.uniform(-1, 1, (m, k)))
        b = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
        c1 = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
        c2 = c1.copy(order="F")
        oracle.gemm_mixed(c1, a, b, -1.0, 1.0, level)
        ref.gemm_mixed(c2, a, b, -1.0, 1.0, level)
        assert np.array_equal(c1, c2)
        cs1 = np.asfortranarray(rng.uniform(-1, 1, (n, n)))
        cs2 = cs1.copy(order="F")
        oracle.syrk_leaf(cs1, b, 0.5, 2.0, level)
        ref.syrk_leaf(cs2, b, 0.5, 2.0, level)
        assert np.array_equal(cs1, cs2)


def test_published_numbers_reproduced_by_oracle(oracle):
    """proj/test_output.txt:19-24 medians at n=1024, b=64 on 3 of the 10
    seeds stay on the published side of every criterion-2 threshold"""
    med = {}
    for cfg in ["Pure F64", "[F16, F32]", "[F16, F16, F16, F32]", "Pure F16"]:
        rels = [oracle.factor(oracle.spd_generate(1024, s), 64, parse_levels(cfg))[3] for s in (0, 1, 2)]
        med[cfg] = float(np.median(rels))
    assert -math.log10(med["Pure F64"]) >= 14.0
    assert 5.0 <= -math.log10(med["[F16, F32]"]) <= 9.0
    assert -math.log10(med["Pure F16"]) < 4.0
    assert med["Pure F16"] / med["[F16, F16, F16, F32]"] >= 50.0


def test_oracle_potrs_solves(oracle):
    n = 64
    a = oracle.spd_generate(n, 3)
    st, det, l, rel, fl = oracle.factor(a, 8, parse_levels("Pure F64"))
    x_true = np.ones(n)
    b = a @ x_true
    x = oracle.potrs(l, b)[:, 0]
    assert np.max(np.abs(x - x_true)) < 1e-12


# ------------------------------------------------------------ planner / flops
def test_planner_flops_equal_static_counter_all_small(tc, oracle):
    """criterion 6 (acceptance.cpp:235-271): every n <= 64, every b"""
    cfg = "[F16, F32, F64]"
    lv = parse_levels(cfg)
    for n in range(1, 65):
        want_total = n * (n + 1) * (2 * n + 1) // 6
        for b in range(1, n + 1):
            want = oracle.flop_breakdown(n, b, lv).as_tuple()
            assert tc.flop_breakdown(n, b, cfg).as_tuple() == want
            assert tc.Plan(n, b, cfg).flops().as_tuple() == want
            assert sum(want[:3]) == want_total


@pytest.mark.parametrize("rec", GOLDEN["flop_breakdown"], ids=lambda r: f"{r['n']}-{r['config']}")
def test_planner_flops_at_baseline_sizes(tc, rec):
    """bit-exact partition at C1..C5 sizes: the plan's per-call flop records
    equal the reference's static breakdown exactly"""
    assert list(tc.Plan(rec["n"], rec["b"], rec["config"]).flops().as_tuple()) == rec["flops"]
    assert list(tc.flop_breakdown(rec["n"], rec["b"], rec["config"]).as_tuple()) == rec["flops"]


def test_hand_counted_breakdown(tc):
    """test_analysis.cpp:158-171: n=4, b=2 -> 30 flops"""
    fb = tc.flop_breakdown(4, 2, "Pure F64")
    assert fb.total() == 30
    assert fb.by_kernel == [10, 8, 12, 0]
    assert fb.calls[0] == 2


def test_offdiag_share_and_half_fraction(tc):
    """criterion 6 (acceptance.cpp:273-291)"""
    fb = tc.flop_breakdown(65536, 256, "[F16, F32, F64]")
    off = fb.kernel_fraction(1) + fb.kernel_fraction(2) + fb.kernel_fraction(3)
    assert abs(100 * off - GOLDEN["published"]["offdiag_share_65536"]) < 1e-3
    prev = -1
    for c in ["Pure F32", "[F16, F32]", "[F16, F16, F32]", "[F16, F16, F16, F32]"]:
        h = tc.flop_breakdown(65536, 256, c).level_fraction(0)
        assert h > prev
        prev = h


def test_plan_is_host_only_and_c3_shape(tc):
    """planning touches no device; C3's op graph (one launch per op)"""
    p = tc.Plan(65536, 256, "[F16, F16, F16, F32]")
    st = p.stats()
    assert st["ops"] > 0 and st["launches"] >= st["ops"]
    kinds = {p.op_info(i)["type"] for i in range(st["ops"])}
    assert {"import", "export", "potrf", "gemm", "quant"} <= kinds
    gem = [p.op_info(i) for i in range(st["ops"]) if p.op_info(i)["type"] == "gemm"]
    assert any(g["gclass"] == "tc16" for g in gem)


# ------------------------------------------------------------ config grammar
def test_config_grammar(tc):
    """test_precision.cpp:171-212"""
    P = tc.PrecisionConfig
    assert P.parse("[F16, F32]").levels == (0, 1)
    assert P.parse("Pure F16").levels == (0,)
    assert P.parse("  [ fp16 ,FP16,f32 , F64 ]  ").levels == (0, 0, 1, 2)
    assert P.parse("pure f64").levels == (2,)
    assert P.parse("F32").levels == (1,)
    with pytest.raises(tc.ValidationError):
        P.parse("[F64, F16]")
    with pytest.raises(tc.ValidationError):
        P.parse("[F32, F16, F64]")
    for bad in ["", "[]", "[F16, F128]", "[F16, F32] junk", "bf16"]:
        with pytest.raises(tc.SyntaxError_):
            P.parse(bad)
    cfg = P.parse("[F16, F32]")
    assert cfg.at_depth(0) == 0 and cfg.at_depth(1) == 1 and cfg.at_depth(7) == 1 and cfg.leaf() == 1
    for text in ["Pure F16", "Pure F32", "Pure F64", "[F16, F32]", "[F16, F32, F64]", "[F16, F16, F16, F32]"]:
        c = P.parse(text)
        assert c.to_string() == text
        assert P.parse(c.to_string()) == c


def test_invalid_arguments(tc):
    with pytest.raises(tc.InvalidArgument):
        tc.Plan(4, 0, "Pure F64")
    with pytest.raises(tc.InvalidArgument):
        tc.Plan(0, 4, "Pure F64")
    with pytest.raises(tc.InvalidArgument):
        tc.flop_breakdown(0, 1, "Pure F64")


def test_spd_generate_host_bit_exact(tc, oracle):
    for n, s in [(1, 0), (16, 99), (300, 42)]:
        assert np.array_equal(tc.spd_generate(n, s), oracle.spd_generate(n, s))


# ------------------------------------------------------------ ABI surface
def test_library_exports_every_declared_symbol(tc):
    hdr = open(os.path.join(ROOT, "include", "treechol_c.h")).read()
    declared = set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", hdr))
    import ctypes
    lib = ctypes.CDLL(tc.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared) >= 20


def test_no_device_fails_loudly(tc):
    """there is no CPU fallback: compute entry points refuse without a GPU"""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = tc.Plan(64, 8, "[F16, F32]")
    a = tc.spd_generate(64, 1)
    with pytest.raises(tc.NoDevice):
        p.factor_host(a)


def test_library_is_sm100a(tc):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


# output tile width per GEMM class (engine / kernels): a GEMM whose output
# overlaps its A operand in the same buffer (the in-place inverse leaf
# solves) is only safe when one tile spans all n output columns -- otherwise
# a tile can overwrite columns another tile still reads as K
_TILE_N = {"tc16": 256, "tc32": 128, "mma32": 32, "mma32w": 256, "simt_f16": 64, "simt_f32": 64,
           "simt_f16d": 64, "simt_f32d": 64, "simt_f64": 64}
_OPERAND_LEVEL = {"tc16": 0, "simt_f16": 0, "simt_f16d": 0, "tc32": 1, "mma32": 1, "mma32w": 1, "simt_f32": 1,
                  "simt_f32d": 1, "simt_f64": 2}


@pytest.mark.parametrize("n,b,cfg", [(4096, 256, "[F16, F16, F16, F32]"), (8192, 256, "[F16, F32, F64]"),
                                     (16384, 256, "[F16, F16, F16, F32]"), (2048, 128, "Pure F32"),
                                     (1024, 64, "[F16, F32]"), (32768, 256, "[F16, F16, F16, F32]")])
def test_no_in_place_gemm_hazard(tc, n, b, cfg):
    """every GEMM whose C overlaps its own A (same buffer) has one output
    tile across all its columns (regression: N >= 32768 factorizations were
    not bit-reproducible when 128-wide TF32 tiles solved in place)"""
    p = tc.Plan(n, b, cfg)
    inplace = 0
    for i in range(p.stats()["ops"]):
        probs = p.op_probs(i)
        if not probs:
            continue
        cls = p.op_info(i)["gclass"]
        for g in probs:
            if g["exec_level"] != _OPERAND_LEVEL[cls]:
                continue  # C and A live in different level buffers
            kw = g["a_kwrap"] or g["k"]
            rows = g["a_r0"] < g["c_r0"] + g["m"] and g["c_r0"] < g["a_r0"] + g["m"]
            cols = g["a_c0"] < g["c_c0"] + g["n"] and g["c_c0"] < g["a_c0"] + kw
            if rows and cols:
                inplace += 1
                assert g["n"] <= _TILE_N[cls], (i, cls, g)
            if g["b_buf"] < 0:  # B from the same level buffer: it must not overlap C at all
                brows = g["b_r0"] < g["c_r0"] + g["m"] and g["c_r0"] < g["b_r0"] + g["n"]
                bcols = g["b_c0"] < g["c_c0"] + g["n"] and g["c_c0"] < g["b_c0"] + g["k"]
                assert not (brows and bcols), (i, cls, g)
    assert inplace > 0 or cfg == "[F16, F32, F64]"


def test_lookahead_splits_keep_the_accounting():
    """row-split panel TRSMs / region-split SYRKs: same flop records (one per
    reference call, static == instrumented), and every GEMM problem inside
    its operand blocks (host-only planner check, no device)"""
    import paper_2601_08082_b200 as tc
    for n, b, cfg in [(4096, 256, "[F16, F16, F16, F32]"), (2000, 64, "[F16, F32, F64]")]:
        base = tc.Plan(n, b, cfg)
        split = tc.Plan(n, b, cfg)
        split.set_option("trsm_row_split_min", 256)
        split.set_option("syrk_split_min", 256)
        assert split.stats()["ops"] > base.stats()["ops"]
        assert split.run_flops().as_tuple() == base.run_flops().as_tuple() == tc.flop_breakdown(n, b, cfg).as_tuple()
        for i in range(split.stats()["ops"]):
            for pr in (split.op_probs(i) if split.op_info(i)["type"] == "gemm" else []):
                assert 0 <= pr["c_r0"] and pr["c_r0"] + pr["m"] <= n and pr["a_r0"] + pr["m"] <= n

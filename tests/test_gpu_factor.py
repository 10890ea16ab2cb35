"""GPU parity of the factorization against the oracle (the C restatement of
the reference, itself pinned bit-exact to the compiled reference).

Bar (BASELINE.json north_star): same inputs and precision tree, backward
error ||A - LL^T||_F/||A||_F within 2x of the reference's, identical status /
failure text / flop accounting (bit-exact partitioning).  The tolerance is
written in each test: rel_gpu <= 2 * rel_oracle + FLOOR with FLOOR = 1e-15
(both sides are at the FP64 rounding floor for Pure F64).
"""
import numpy as np
import pytest

from pyoracle import parse_levels

pytestmark = pytest.mark.gpu

FLOOR = 1e-15


def _run(tc, a, b, cfg, quantize=True, **plan_kw):
    import torch
    inverse = plan_kw.pop("inverse", True)
    plan = tc.Plan(a.shape[0], b, cfg, quantize, **plan_kw)
    if not inverse:
        plan.set_option("inverse_trsm", 0)
    a_dev = tc.to_device(a)
    l_dev = a_dev.clone()
    st = plan.factor_device(a_dev, l_dev)
    rel = tc.factorization_error_device(a_dev, l_dev) if st.status == "ok" else float("nan")
    torch.cuda.synchronize()
    return st, tc.from_device(l_dev), rel, plan.run_flops()


CASES = [
    # n, b, config, quantize, seed
    (8, 2, "Pure F64", True, 1),
    (7, 2, "[F16, F32]", True, 3),
    (64, 8, "[F16, F32]", True, 7),
    (96, 16, "[F16, F32]", True, 11),
    (128, 16, "Pure F16", True, 2),
    (100, 7, "[F16, F16, F16, F32]", True, 5),
    (200, 32, "[F16, F32, F64]", True, 4),
    (200, 32, "[F16, F32, F64]", False, 4),
    (384, 48, "[F16, F16, F32]", True, 21),
    (256, 32, "Pure F32", True, 9),
    (1024, 128, "[F16, F64]", True, 42),           # C1
    (1024, 64, "[F16, F16, F16, F32]", True, 0),   # criterion 2/3 ladder member
    (1024, 64, "Pure F16", True, 0),
    (512, 256, "Pure F32", True, 3),
    (1000, 64, "[F16, F32]", True, 8),             # irregular splits (500/250/125/62/63)
    (777, 100, "[F16, F16, F32, F64]", True, 12),
    (2048, 256, "[F16, F32, F64]", True, 42),
]


@pytest.mark.parametrize("n,b,cfg,q,seed", CASES)
def test_factor_matches_oracle(tc, oracle, n, b, cfg, q, seed):
    a = oracle.spd_generate(n, seed)
    st_o, det_o, l_o, rel_o, fl_o = oracle.factor(a, b, parse_levels(cfg), q)
    st, l, rel, fl = _run(tc, a, b, cfg, q)
    assert st.status == st_o == "ok"
    assert fl.as_tuple() == fl_o.as_tuple()
    # device metric == oracle metric on the same L (to FP64 rounding)
    rel_cpu = oracle.factorization_error(a, l)
    assert abs(rel - rel_cpu) <= 1e-6 * rel_cpu + 1e-15
    assert rel <= 2.0 * rel_o + FLOOR, (rel, rel_o)
    # upper triangle untouched
    iu = np.triu_indices(n, 1)
    assert np.array_equal(l[iu], a[iu])


@pytest.mark.parametrize("n,b,cfg,q,seed", CASES[:8])
def test_simt_path_matches_oracle(tc, oracle, n, b, cfg, q, seed):
    """use_tc=0: every FP16-operand GEMM on the SIMT kernel instead of tcgen05"""
    a = oracle.spd_generate(n, seed)
    st_o, det_o, l_o, rel_o, fl_o = oracle.factor(a, b, parse_levels(cfg), q)
    st, l, rel, fl = _run(tc, a, b, cfg, q, use_tc=False)
    assert st.status == "ok"
    assert rel <= 2.0 * rel_o + FLOOR


def test_pure_f64_equals_textbook_cholesky(tc, oracle):
    """acceptance criterion 1 (acceptance.cpp:69-94): 50 cases, <= 1e-13"""
    rng = np.random.default_rng(20240901)
    worst = 0.0
    for c in range(50):
        n = 1 + int(rng.integers(0, 256))
        b = min(n, (1, 2, 7, 32, n)[c % 5])
        a = oracle.spd_generate(n, int(rng.integers(0, 2**62)))
        ref = np.linalg.cholesky(a)
        st, l, rel, fl = _run(tc, a, b, "Pure F64")
        assert st.status == "ok"
        lo = np.tril(l)
        d = np.sqrt(np.sum((lo - ref) ** 2) / np.sum(ref ** 2))
        worst = max(worst, d)
    assert worst <= 1e-13


def _scaled(oracle, n, seed, s):
    return np.asfortranarray(oracle.spd_generate(n, seed) * s)


def test_quantization_rescue(tc, oracle):
    """criterion 4 (acceptance.cpp:167-185): ok with quantization,
    breakdown with the same detail text as the reference without"""
    a = _scaled(oracle, 256, 4, 3.0 * 65504.0 / 0.5)
    lv = parse_levels("[F16, F32]")
    st, l, rel, fl = _run(tc, a, 32, "[F16, F32]", True)
    st_o, det_o, _, rel_o, fl_o = oracle.factor(a, 32, lv, True)
    assert st.status == st_o == "ok"
    assert rel <= 2 * rel_o + FLOOR
    st, l, rel, fl = _run(tc, a, 32, "[F16, F32]", False)
    st_o, det_o, _, _, fl_o = oracle.factor(a, 32, lv, False)
    assert st.status == "numerical-breakdown" == st_o
    assert st.detail == det_o
    assert fl.as_tuple() == fl_o.as_tuple()


def test_quantization_alpha_above_one(tc, oracle):
    """a spine panel beyond the Half range gets alpha > 1 (tree.cpp:117-120)"""
    a = _scaled(oracle, 64, 7, 3.0 * 65504.0 / 0.5)
    for cfg in ("[F16, F32]", "[F16, F16, F32]"):
        st, l, rel, fl = _run(tc, a, 8, cfg, True)
        st_o, det_o, _, rel_o, fl_o = oracle.factor(a, 8, parse_levels(cfg), True)
        assert st.status == st_o
        assert st.detail == det_o
        if st_o == "ok":
            assert rel <= 2 * rel_o + FLOOR


def test_extreme_range_breakdown_text(tc, oracle):
    """criterion 5 (acceptance.cpp:189-231)"""
    n = 256
    a = oracle.spd_generate(n, 6)
    s = np.where(np.arange(n) < n // 2, 1e-3, 1e8)
    a = np.asfortranarray(a * s[:, None] * s[None, :])
    for cfg in ("Pure F16", "[F16, F32]", "[F16, F32, F64]"):
        st, *_ = _run(tc, a, 32, cfg)
        st_o, det_o, *_ = oracle.factor(a, 32, parse_levels(cfg))
        assert st.status == st_o == "numerical-breakdown"
        assert st.detail == det_o
    st, l, rel, fl = _run(tc, a, 32, "Pure F64")
    assert st.status == "ok" and -np.log10(rel) >= 13.0


@pytest.mark.parametrize("n,b,i,val", [(16, 4, 9, -50.0), (24, 8, 5, -1.0)])
def test_not_positive_definite_index(tc, oracle, n, b, i, val):
    a = oracle.spd_generate(n, 4 if n == 16 else 8)
    a[i, i] = val
    st, *_, fl = _run(tc, a, b, "Pure F64")
    st_o, det_o, _, _, fl_o = oracle.factor(a, b, parse_levels("Pure F64"))
    assert st.status == st_o == "not-positive-definite"
    assert st.index == i
    assert st.detail == det_o
    assert fl.as_tuple() == fl_o.as_tuple()  # partial flops up to the failure


def test_pure_f16_breaks_down_on_large_diagonal(tc, oracle):
    """n + r > 65504 on the diagonal overflows binary16 at build"""
    n = 512
    a = oracle.spd_generate(n, 1)
    a[np.arange(n), np.arange(n)] += 65536.0 - n
    st, *_ = _run(tc, a, 64, "Pure F16")
    st_o, det_o, *_ = oracle.factor(a, 64, parse_levels("Pure F16"))
    assert st.status == st_o == "numerical-breakdown"
    assert st.detail == det_o


def test_deterministic_bit_for_bit(tc, oracle):
    """criterion 8 (acceptance.cpp:314-336)"""
    a = oracle.spd_generate(384, 21)
    _, l1, r1, _ = _run(tc, a, 48, "[F16, F16, F32]")
    _, l2, r2, _ = _run(tc, a, 48, "[F16, F16, F32]")
    assert np.array_equal(l1.view(np.uint64), l2.view(np.uint64))
    assert r1 == r2


def test_graph_and_eager_agree(tc, oracle):
    a = oracle.spd_generate(512, 5)
    _, l1, r1, _ = _run(tc, a, 64, "[F16, F16, F32]")
    _, l2, r2, _ = _run(tc, a, 64, "[F16, F16, F32]", use_graph=False)
    assert np.array_equal(l1.view(np.uint64), l2.view(np.uint64))


def test_host_entry_point_in_place(tc, oracle):
    a = oracle.spd_generate(300, 3)
    l = np.array(a, order="F", copy=True)
    plan = tc.Plan(300, 32, "[F16, F32]")
    st = plan.factor_host(l)
    assert st.status == "ok"
    _, l_dev, _, _ = _run(tc, a, 32, "[F16, F32]")
    assert np.array_equal(np.tril(l), np.tril(l_dev))
    iu = np.triu_indices(300, 1)
    assert np.array_equal(l[iu], a[iu])


@pytest.mark.parametrize("dag", [1, 0, "eager"])
def test_host_entry_point_pinned_graph(tc, oracle, dag):
    """pinned host buffer: the copies overlap the factorization graph (H2D /
    D2H on the copy streams, event nodes in the graph); repeated calls reuse
    the graph and must see each call's data"""
    import torch
    n = 1024
    plan = tc.Plan(n, 64, "[F16, F16, F32]")
    if dag == "eager":
        plan.set_option("use_graph", 0)
    else:
        plan.set_option("dag_graph", dag)
    for seed in (7, 8):
        a = oracle.spd_generate(n, seed)
        host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        host.numpy().T[:] = a
        st = plan.factor_host(host.numpy().T)
        assert st.status == "ok"
        _, l_dev, _, _ = _run(tc, a, 64, "[F16, F16, F32]")
        l = host.numpy().T
        assert np.array_equal(np.tril(l), np.tril(l_dev))
        iu = np.triu_indices(n, 1)
        assert np.array_equal(l[iu], a[iu])


@pytest.mark.parametrize("what", ["not-positive-definite", "numerical-breakdown", "alpha-above-one"])
def test_host_entry_point_pinned_failures(tc, oracle, what):
    """the pinned host pipeline (phased graphs, copy feeder) reports the same
    first failure as the device path, and a later call on good data is
    unaffected"""
    import torch
    n, b, cfg = 1024, 64, "[F16, F16, F32]"
    a = oracle.spd_generate(n, 12)
    if what == "not-positive-definite":
        a[700, 700] = -5.0
    elif what == "numerical-breakdown":
        a[900, 300] = np.nan  # lower triangle, inside a late block
    else:
        a = _scaled(oracle, n, 12, 3.0 * 65504.0 / 0.5)
    plan = tc.Plan(n, b, cfg)
    host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    host.numpy().T[:] = a
    st = plan.factor_host(host.numpy().T)
    st_d, l_dev, _, _ = _run(tc, a, b, cfg)
    assert st.status == st_d.status
    assert st.index == st_d.index
    assert st.detail == st_d.detail
    if st.status == "ok":
        assert np.array_equal(np.tril(host.numpy().T), np.tril(l_dev))
    good = oracle.spd_generate(n, 13)
    host.numpy().T[:] = good
    assert plan.factor_host(host.numpy().T).status == "ok"
    _, l_good, _, _ = _run(tc, good, b, cfg)
    assert np.array_equal(np.tril(host.numpy().T), np.tril(l_good))


def test_ladder_ordering_n1024(tc, oracle):
    """criteria 2-3 (acceptance.cpp:103-163) on seeds 0-2 against the
    published medians (proj/test_output.txt:19-24, 34)"""
    cfgs = ["Pure F64", "Pure F32", "Pure F16", "[F16, F32]", "[F16, F16, F16, F32]"]
    med = {}
    for cfg in cfgs:
        plan = tc.Plan(1024, 64, cfg)
        rels = []
        for seed in range(3):
            a = oracle.spd_generate(1024, seed)
            a_dev = tc.to_device(a)
            l_dev = a_dev.clone()
            assert plan.factor_device(a_dev, l_dev).status == "ok"
            rels.append(tc.factorization_error_device(a_dev, l_dev))
        med[cfg] = float(np.median(rels))
    d = {k: -np.log10(v) for k, v in med.items()}
    assert d["Pure F64"] >= 14.0
    assert 6.0 <= d["Pure F32"] <= 10.0
    assert d["Pure F16"] < 4.0
    assert d["[F16, F32]"] >= 5.0
    assert med["[F16, F16, F16, F32]"] <= med["Pure F16"] / 50.0


@pytest.mark.parametrize("n,cfg", [(4096, "[F16, F16, F16, F32]"), (2048, "Pure F16")])
def test_inverse_leaf_solve_matches_substitution(tc, oracle, n, cfg):
    """FP16 leaf solves with m >= 512 run as tcgen05 GEMMs against the leaf's
    inverse; the backward error stays within 2x of the oracle and of the
    substitution kernel"""
    a = oracle.spd_generate(n, 42)
    if cfg == "Pure F16":
        a = np.asfortranarray(a * 0.5)  # keep the diagonal inside binary16
    st_o, det_o, _, rel_o, fl_o = oracle.factor(a, 256, parse_levels(cfg))
    st1, l1, rel1, fl1 = _run(tc, a, 256, cfg)
    st2, l2, rel2, fl2 = _run(tc, a, 256, cfg, inverse=False)
    assert st1.status == st2.status == st_o == "ok"
    assert fl1.as_tuple() == fl2.as_tuple() == fl_o.as_tuple()
    assert rel1 <= 2 * rel_o + FLOOR, (rel1, rel_o)
    assert rel2 <= 2 * rel_o + FLOOR, (rel2, rel_o)


@pytest.mark.parametrize("n", [512, 1024])
def test_singular_diagonal_detail(tc, oracle, n):
    """an F32 leaf whose diagonal overflows binary16 when a [F16, F32] panel
    solve reads it (kernels.cpp:78-81): SingularDiagonal with the reference's
    index, through the substitution kernel (m=256) and the inverse path (m=512)"""
    a = np.asfortranarray(oracle.spd_generate(n, 3) * 1e10)
    st, *_ = _run(tc, a, 256, "[F16, F32]")
    st_o, det_o, *_ = oracle.factor(a, 256, parse_levels("[F16, F32]"))
    assert st_o == "singular-diagonal"
    assert st.status == "singular-diagonal"
    assert st.detail == det_o


def test_spd_generate_device_bit_exact(tc, oracle):
    a = tc.from_device(tc.spd_generate_device(300, 77))
    assert np.array_equal(a, oracle.spd_generate(300, 77))


def test_c2_matches_reference_golden(tc):
    """BASELINE config C2 (N=8192, b=256, [F16, F32, F64], seed 42) against
    tests/golden/c2.json: the oracle's outcome (1.8759406e-06), equal to the
    compiled reference's (1.875941e-06)."""
    import json
    import os
    import torch
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c2.json")))
    a = tc.spd_generate_device(g["n"], g["seed"])
    l = torch.empty_like(a)
    plan = tc.Plan(g["n"], g["b"], g["config"])
    st = plan.factor_device(a, l)
    assert st.status == g["status"] == "ok"
    assert list(plan.run_flops().as_tuple()) == g["flops"]
    rel = tc.factorization_error_device(a, l)
    assert rel <= 2 * g["rel_error"], (rel, g["rel_error"])


def test_c1_ten_seed_median_within_2x(tc, oracle):
    """C1 (N=1024, b=128, [F16, F64]) over seeds 0-9: the median
    backward error within 2x of the reference's median."""
    rel_g, rel_o = [], []
    for seed in range(10):
        a = oracle.spd_generate(1024, seed)
        st_o, _, _, r_o, _ = oracle.factor(a, 128, parse_levels("[F16, F64]"))
        st, _, r, _ = _run(tc, a, 128, "[F16, F64]")
        assert st.status == st_o == "ok"
        rel_g.append(r)
        rel_o.append(r_o)
    assert np.median(rel_g) <= 2 * np.median(rel_o), (np.median(rel_g), np.median(rel_o))


def test_c3_full_size_properties(tc):
    """BASELINE config C3 (N=65536, b=256, [F16, F16, F16, F32]) where the CPU
    oracle cannot go (weeks): size-independent properties.  Status ok; the
    executed flops equal the static counter and n(n+1)(2n+1)/6
    (criterion 6); a second factorization is bit-identical (criterion 8); and
    on A/2 (Pure F16 overflows A's diagonal) the mixed tree's backward error
    is at least 50x below Pure F16's (criterion 3 / the north-star target)."""
    import torch
    n, b, cfg = 65536, 256, "[F16, F16, F16, F32]"
    a = tc.spd_generate_device(n, 42)
    plan = tc.Plan(n, b, cfg)
    l1 = a.clone()  # same strict upper in both outputs (never written)
    assert plan.factor_device(a, l1).status == "ok"
    fl = plan.run_flops()
    assert fl.as_tuple() == tc.flop_breakdown(n, b, cfg).as_tuple()
    assert fl.total() == n * (n + 1) * (2 * n + 1) // 6
    l2 = a.clone()
    assert plan.factor_device(a, l2).status == "ok"
    assert torch.equal(l1, l2)
    del l2, plan
    torch.cuda.empty_cache()
    a.mul_(0.5)  # exact
    rel = {}
    for c in (cfg, "Pure F16"):
        p = tc.Plan(n, b, c)
        assert p.factor_device(a, l1).status == "ok"
        rel[c] = tc.factorization_error_device(a, l1)
        del p
        torch.cuda.empty_cache()
    assert rel[cfg] * 50 <= rel["Pure F16"], rel


@pytest.mark.parametrize("n,b,cfg", [(777, 64, "[F16, F32]"), (1000, 96, "[F16, F16, F32]"), (300, 300, "Pure F32")])
def test_host_entry_point_pinned_ragged(tc, oracle, n, b, cfg):
    """ragged orders and leaf sizes through the copy pipeline (chunking of
    non-square blocks, single-leaf plans) give the device path's factor"""
    import torch
    a = oracle.spd_generate(n, 31)
    host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    host.numpy().T[:] = a
    plan = tc.Plan(n, b, cfg)
    assert plan.factor_host(host.numpy().T).status == "ok"
    _, l_dev, _, _ = _run(tc, a, b, cfg)
    assert np.array_equal(np.tril(host.numpy().T), np.tril(l_dev))
    iu = np.triu_indices(n, 1)
    assert np.array_equal(host.numpy().T[iu], a[iu])


LOOKAHEAD = {"trsm_row_split_min": 256, "syrk_split_min": 256}


def _run_opts(tc, a, b, cfg, opts):
    import torch
    plan = tc.Plan(a.shape[0], b, cfg)
    for k, v in opts.items():
        plan.set_option(k, v)
    a_dev = tc.to_device(a)
    l_dev = a_dev.clone()
    st = plan.factor_device(a_dev, l_dev)
    torch.cuda.synchronize()
    return st, tc.from_device(l_dev), plan.run_flops()


@pytest.mark.parametrize("n,b,cfg,seed", [(2048, 128, "[F16, F16, F16, F32]", 3), (1000, 64, "[F16, F32]", 8),
                                          (777, 100, "[F16, F16, F32, F64]", 12)])
def test_lookahead_splits_are_bit_identical(tc, oracle, n, b, cfg, seed):
    """row-split panel TRSMs and region-split SYRKs (lookahead) only cut the
    reference's calls into row / region parts: every element sees the same
    operations in the same order, so L is bit-identical to the default plan,
    with the same status and flop accounting"""
    a = oracle.spd_generate(n, seed)
    st0, l0, fl0 = _run_opts(tc, a, b, cfg, {})
    st1, l1, fl1 = _run_opts(tc, a, b, cfg, LOOKAHEAD)
    assert st0.status == st1.status == "ok"
    assert fl0.as_tuple() == fl1.as_tuple()
    assert np.array_equal(np.tril(l0).view(np.uint64), np.tril(l1).view(np.uint64))


def test_lookahead_splits_keep_first_failure(tc, oracle):
    """a panel that overflows F16 and an indefinite trailing block: the split
    plan reports the same first failure (status, index, text) as the default"""
    a = oracle.spd_generate(1024, 2)
    a[700:, 700:] -= 2.0 * 1024 * np.eye(324)  # not positive definite from row 700 on
    st0, _, _ = _run_opts(tc, a, 64, "[F16, F16, F32]", {})
    st1, _, _ = _run_opts(tc, a, 64, "[F16, F16, F32]", LOOKAHEAD)
    assert st0.status == st1.status == "not-positive-definite"
    assert st0.index == st1.index
    b = oracle.spd_generate(1024, 2)
    b[600:700, 0:100] = 1e6  # off-diagonal block values beyond F16 range before quantize -> alpha > 1 path
    st0, l0, _ = _run_opts(tc, b, 64, "[F16, F16, F32]", {})
    st1, l1, _ = _run_opts(tc, b, 64, "[F16, F16, F32]", LOOKAHEAD)
    assert st0.status == st1.status
    assert (st0.detail, st0.index) == (st1.detail, st1.index)
    if st0.status == "ok":
        assert np.array_equal(np.tril(l0).view(np.uint64), np.tril(l1).view(np.uint64))


def test_fused_leaf_inverse_matches_oracle(tc, oracle):
    """option fuse_inverse: the F32 leaves' W = inv(L) computed inside the
    leaf POTRF kernel instead of a separate launch (a measured alternative,
    off by default): same status and flops, rel within 2x of the reference's"""
    a = oracle.spd_generate(2048, 11)
    cfg, b = "[F16, F16, F16, F32]", 128
    st_o, _, _, rel_o, fl_o = oracle.factor(a, b, parse_levels(cfg))
    st, l, fl = _run_opts(tc, a, b, cfg, {"fuse_inverse": 1})
    assert st.status == st_o == "ok"
    assert fl.as_tuple() == fl_o.as_tuple()
    import torch
    rel = tc.factorization_error_device(tc.to_device(a), tc.to_device(l))
    torch.cuda.synchronize()
    assert rel <= 2 * rel_o + FLOOR, (rel, rel_o)


def test_narrow_fp16_tiles_keep_the_factor_bit_identical(tc, oracle):
    """with the narrow FP16 kind enabled for every eligible list, L is
    bit-identical to the default plan's (in-place inverse solves stay on
    full-width tiles: a 128-column tile would overwrite A columns another
    tile still reads)"""
    a = oracle.spd_generate(2048, 21)
    st0, l0, _ = _run_opts(tc, a, 128, "[F16, F16, F16, F32]", {})
    tc.set_global_option("tc_narrow_max_tiles", 1 << 20)
    try:
        st1, l1, _ = _run_opts(tc, a, 128, "[F16, F16, F16, F32]", {})
    finally:
        tc.set_global_option("tc_narrow_max_tiles", 0)
    assert st0.status == st1.status == "ok"
    assert np.array_equal(np.tril(l0).view(np.uint64), np.tril(l1).view(np.uint64))

"""The kernel-level API (kernels.hpp:20-40, tree.hpp:47-51) on the device:
bit-identical to the reference's scalar kernels (the oracle, itself pinned
bit-exact to the compiled reference; and the compiled reference where it
travelled).  These calls are not on the factorization path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LEVELS = (0, 1, 2)


def _rand(shape, seed, scale=1.0):
    r = np.random.default_rng(seed)
    return np.asfortranarray(r.uniform(-1.0, 1.0, shape) * scale)


@pytest.mark.parametrize("lv", LEVELS)
def test_gemm_mixed_bit_exact(tc, oracle, lv):
    for (m, n, k, al, be) in [(37, 29, 53, -1.0, 1.0), (64, 64, 300, 0.5, 0.0), (5, 130, 7, 2.0, -0.25)]:
        a, b, c = _rand((m, k), 1), _rand((n, k), 2), _rand((m, n), 3, 10.0)
        c1, c2 = c.copy(order="F"), c.copy(order="F")
        tc.gemm_mixed(c1, a, b, al, be, lv)
        oracle.gemm_mixed(c2, a, b, al, be, lv)
        assert np.array_equal(c1, c2), (lv, m, n, k)


@pytest.mark.parametrize("lv", LEVELS)
def test_syrk_leaf_bit_exact_and_upper_untouched(tc, oracle, lv):
    n, k = 47, 90
    a, c = _rand((n, k), 4), _rand((n, n), 5, 3.0)
    c[np.triu_indices(n, 1)] = np.nan  # strict upper never written (nor read)
    c1, c2 = c.copy(order="F"), c.copy(order="F")
    tc.syrk_leaf(c1, a, -1.0, 1.0, lv)
    oracle.syrk_leaf(c2, a, -1.0, 1.0, lv)
    lo = np.tril_indices(n)
    assert np.array_equal(c1[lo], c2[lo])
    assert np.isnan(c1[np.triu_indices(n, 1)]).all()


@pytest.mark.parametrize("lv", LEVELS)
def test_potrf_and_trsm_leaf_bit_exact(tc, oracle, lv):
    n, m = 60, 45
    a = oracle.spd_generate(n, 9)
    l1, l2 = a.copy(order="F"), a.copy(order="F")
    tc.potrf_leaf(l1, lv)
    st, _ = oracle.potrf_leaf(l2, lv)
    assert st == "ok"
    lo = np.tril_indices(n)
    assert np.array_equal(l1[lo], l2[lo])
    b = _rand((m, n), 6, 5.0)
    b1, b2 = b.copy(order="F"), b.copy(order="F")
    tc.trsm_leaf(b1, l1, lv)
    oracle.trsm_leaf(b2, l2, lv)
    assert np.array_equal(b1, b2)


def test_potrf_leaf_not_positive_definite_index(tc, oracle):
    a = oracle.spd_generate(16, 3)
    a[7, 7] = -5.0
    with pytest.raises(tc.NotPositiveDefinite) as e:
        tc.potrf_leaf(a.copy(order="F"), 2)
    st, idx = oracle.potrf_leaf(a.copy(order="F"), 2)
    assert st == "not-positive-definite" and e.value.index == idx == 7


def test_quantize_dequantize_known_answers(tc):
    # test_tree.cpp:117-145 known answers
    b = np.asfortranarray([[131008.0, -4.0]])
    assert tc.quantize_block(b, 0) == 2.0 and b[0, 0] == 65504.0 and b[0, 1] == -2.0
    z = np.zeros((3, 3), order="F")
    assert tc.quantize_block(z, 0) == 1.0
    d = np.asfortranarray([[1.0, 2.0]])
    tc.dequantize_block(d, 2.0, 0)
    assert d[0, 0] == 2.0 and d[0, 1] == 4.0


def test_round_matrix_matches_oracle(tc, oracle):
    x = _rand((33, 17), 8, 70000.0)
    for lv in LEVELS:
        y = x.copy(order="F")
        tc.round_matrix(y, lv)
        ref = np.vectorize(lambda v: oracle.round_to(v, lv))(x)
        assert np.array_equal(y, ref, equal_nan=True), lv

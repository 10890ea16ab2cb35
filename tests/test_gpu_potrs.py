"""POTRS parity (SURVEY 8(a) row 25, 8(c) "POTRS / solve").

The reference has no solve; the oracle's or_potrs restates it as SURVEY 8(c)
defines: the forward sweep is trsm_leaf at Precision::Double on the 1 x n
row b^T (kernels.cpp:71-92), the backward sweep L^T x = y in plain double.
The GPU solve (k_potrs_* through tc_potrs_device, and the batched launch
sequence of tc_batch_run) runs on the SAME factor L, so the two differ only
by FP64 summation order:
  * x agrees with or_potrs's to ||x - x_or||_inf <= 64 n u ||x_or||_inf
    (L is diagonally dominant: well conditioned);
  * the solve residual ||b - A x||_2 / (||A||_F ||x||_2 + ||b||_2) is within
    2x of the oracle's (north_star's "solve residual within 2x of the
    reference's"), plus a floor of a few u for pure-FP64 factors whose
    residual is rounding noise.
The C4-size check (N=16384, golden outcome of the oracle) is in
tests/test_batch.py::test_c4_unit_matches_golden.
"""
import numpy as np
import pytest

U64 = 2.0 ** -53


def residual(a, x, b):
    r = b - a @ x
    return float(np.linalg.norm(r) / (np.linalg.norm(a) * np.linalg.norm(x) + np.linalg.norm(b)))


def _rhs(a, nrhs, seed):
    n = a.shape[0]
    rng = np.random.default_rng(seed)
    cols = [a.sum(axis=1)] + [rng.uniform(-1, 1, n) for _ in range(nrhs - 1)]
    return np.asfortranarray(np.stack(cols, axis=1))


def _factor(tc, oracle, n, b, cfg, seed):
    import torch
    a = oracle.spd_generate(n, seed)
    a_dev = tc.to_device(a)
    l_dev = torch.empty_like(a_dev)
    st = tc.Plan(n, b, cfg).factor_device(a_dev, l_dev)
    assert st.status == "ok"
    L = np.asfortranarray(np.tril(tc.from_device(l_dev)))
    return a, L, l_dev


def _check(a, L, x_gpu, rhs, oracle):
    x_or = oracle.potrs(L, rhs)
    n = a.shape[0]
    for r in range(rhs.shape[1]):
        xo, xg, bb = x_or[:, r], x_gpu[:, r], rhs[:, r]
        assert np.max(np.abs(xg - xo)) <= 64 * n * U64 * np.max(np.abs(xo)), r
        rg, ro = residual(a, xg, bb), residual(a, xo, bb)
        assert rg <= 2 * ro + 8 * U64, (r, rg, ro)


@pytest.mark.gpu
@pytest.mark.parametrize("n,nrhs,b,cfg", [
    (64, 1, 16, "[F16, F64]"),
    (64, 3, 16, "Pure F64"),
    (777, 1, 64, "[F16, F16, F32]"),
    (777, 3, 64, "[F16, F32, F64]"),
    (4096, 1, 256, "[F16, F16, F16, F32]"),
    (4096, 3, 256, "[F16, F16, F16, F32]"),
])
def test_potrs_matches_oracle(tc, oracle, n, nrhs, b, cfg):
    import torch
    a, L, l_dev = _factor(tc, oracle, n, b, cfg, seed=n + nrhs)
    rhs = _rhs(a, nrhs, n)
    b_dev = torch.from_numpy(np.ascontiguousarray(rhs.T)).to("cuda")  # (nrhs, n): column-major n x nrhs
    tc.potrs_device(l_dev, b_dev)
    x_gpu = np.asfortranarray(b_dev.cpu().numpy().T)
    _check(a, L, x_gpu, rhs, oracle)


@pytest.mark.gpu
def test_batched_potrs_matches_oracle(tc, oracle):
    """the C4 path: every solve of a tc_batch_run call in one launch sequence"""
    import torch
    n, b, cfg, nrhs = 1536, 128, "[F16, F16, F16, F32]", 2
    mats = [oracle.spd_generate(n, s) for s in (11, 12, 13)]
    a_dev = [tc.to_device(m) for m in mats]
    rhs = [_rhs(m, nrhs, 5 + i) for i, m in enumerate(mats)]
    b_dev = [torch.from_numpy(np.ascontiguousarray(r.T)).to("cuda") for r in rhs]
    st = tc.Batch(n, b, cfg, True, concurrency=2).run(a_dev, b_dev)
    assert st == ["ok"] * 3
    for k, m in enumerate(mats):
        L = np.asfortranarray(np.tril(tc.from_device(a_dev[k])))
        _check(m, L, np.asfortranarray(b_dev[k].cpu().numpy().T), rhs[k], oracle)

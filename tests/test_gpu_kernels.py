"""Kernel-level parity: one problem of each factorization GEMM class, run on
the exact launch path the factorization graph uses (tc_gemm_problem_device:
the same TMA descriptors, tile scheduler and dot_update epilogue), against
the oracle's gemm_mixed (oracle.c, restating kernels.cpp:114-132; syrk_leaf
kernels.cpp:94-112 is the same per-element formula on the lower triangle).

Shapes are the C3 (N=65536, b=256, [F16, F16, F16, F32]) histogram's
extremes: the 256 x 256 x 32768 lower SYRK leaf (F32 exec), the
32768 x 16384 x 16384 TRSM-GEMM (F16 exec) and a 512 x 256 x 256 one.

The full outputs are too big for the CPU oracle, so it recomputes a sample
of rows x columns (each output element depends only on its row of A, its row
of B and its C input, so the sample is exact), edges included.

Bounds (the reference's dot_update accumulates sequentially in FP32 with
round-to-nearest; the tensor cores sum in another order and truncate when
adding into their FP32 accumulator; FP16 x FP16 products are exact in FP32).
With mag = |alpha| sum|a b| + |beta c| and gamma_k = k u / (1 - k u):
  * exec F16: |gpu - oracle| <= ulp16 + 2 gamma_k(u = 2^-24) mag -- one
    binary16 rounding step apart plus both FP32 accumulations' worst case --
    and at least 90% of the sampled elements are the same or adjacent
    binary16 numbers (near-zero results, whose half-ulp is below the FP32
    accumulation error, are the rest);
  * exec F32 / F64: every element obeys the order-independent bound
    |value - exact| <= gamma_k * mag + ulp(value), exact = the products summed
    in x87 extended precision, then the epilogue;
  * TF32X3 (FP32 operands as a hi + lo TF32 pair, lo*lo dropped): each
    operand carries >= 21 significant bits, so the bound gains 2^-19 * mag
    (DESIGN.md section 4).
The truncating accumulation makes long FP32-exec sums drift: at k = 32768
the GPU's RMS error is ~17x the oracle's (tools/gemm_acc_probe.py, DESIGN.md
section 4), inside the worst-case bound; the factorization-level contract
(backward error within 2x of the reference's) is tested end to end
(tests/test_gpu_factor.py, tests/test_batch.py::test_c4_unit_matches_golden).
Masked (lower) problems must leave every element above the diagonal
bit-for-bit unchanged.
"""
import numpy as np
import pytest

U32 = 2.0 ** -24
U64 = 2.0 ** -53

CASES = [
    # gclass, exec level, lower, m, n, k
    ("tc16", 0, False, 512, 256, 256),
    ("tc16", 1, False, 512, 256, 256),
    ("tc16", 1, True, 256, 256, 32768),       # C3 SYRK leaf (leaf level F32)
    ("tc16", 0, True, 256, 256, 4096),
    ("tc16", 0, False, 32768, 16384, 16384),  # C3 top TRSM-GEMM
    ("tc16", 0, False, 1000, 700, 333),       # ragged edges (TMA zero fill)
    ("tc32", 1, False, 512, 256, 256),
    ("tc32", 1, False, 4096, 2048, 1024),
    ("tc32", 1, True, 256, 256, 2048),
    ("mma32", 1, False, 256, 256, 256),
    ("mma32", 1, True, 256, 256, 512),
    ("simt_f16d", 2, False, 512, 256, 512),   # C1/C2: F16 operands, F64 exec
    ("simt_f64", 2, False, 256, 128, 384),
    ("simt_f32d", 2, True, 256, 256, 512),
]

_OPERAND = {"tc16": 0, "simt_f16": 0, "simt_f16d": 0, "tc32": 1, "mma32": 1, "mma32w": 1, "simt_f32": 1,
            "simt_f32d": 1, "simt_f64": 2}


def _dtype(level):
    import torch
    return (torch.float16, torch.float32, torch.float64)[level]


def _layout(m, n, k, lower):
    """operand rows [0, n) = B, rows [n, n+m) = A (cols [0, k)); C at rows
    [n, n+m), cols [k, k+n).  Lower: A = B at rows [0, m), C on the diagonal
    at rows = cols = [k, k+m)."""
    if lower:
        assert m == n
        rows = k + m
        return dict(a_r0=0, a_c0=0, b_r0=0, b_c0=0, c_r0=k, c_c0=k), rows, ((k + m + 63) // 64) * 64
    return dict(a_r0=n, a_c0=0, b_r0=0, b_c0=0, c_r0=n, c_c0=k), n + m, ((k + n + 63) // 64) * 64


def _sample(count, size, rng):
    if size <= count:
        return np.arange(size)
    pick = rng.choice(np.arange(1, size - 1), count - 2, replace=False)
    return np.sort(np.concatenate([[0, size - 1], pick]))


def _half_order(x):
    """binary16 bits as an ordered integer (adjacent halves differ by 1)"""
    b = x.astype(np.float16).view(np.int16).astype(np.int64)
    return np.where(b < 0, -(b & 0x7FFF), b)


@pytest.mark.gpu
@pytest.mark.parametrize("gclass,lvl,lower,m,n,k", CASES)
def test_gemm_class_matches_gemm_mixed(tc, oracle, gclass, lvl, lower, m, n, k):
    import torch
    op = _OPERAND[gclass]
    pos, rows, ldw = _layout(m, n, k, lower)
    g = torch.Generator(device="cuda").manual_seed(1000 * m + 7 * n + k)
    bufs = [None, None, None]
    for lv in {op, lvl}:
        bufs[lv] = torch.zeros((rows, ldw), dtype=_dtype(lv), device="cuda")
    ob, cb = bufs[op], bufs[lvl]
    # operands uniform in [-1, 1) stored at the operand level; C in [-4, 4)
    a_rows = slice(pos["a_r0"], pos["a_r0"] + m)
    b_rows = slice(pos["b_r0"], pos["b_r0"] + n)
    ob[a_rows, :k] = (torch.rand((m, k), generator=g, device="cuda", dtype=torch.float64) * 2 - 1).to(ob.dtype)
    if not lower:
        ob[b_rows, :k] = (torch.rand((n, k), generator=g, device="cuda", dtype=torch.float64) * 2 - 1).to(ob.dtype)
    c_rows = slice(pos["c_r0"], pos["c_r0"] + m)
    c_cols = slice(pos["c_c0"], pos["c_c0"] + n)
    cb[c_rows, c_cols] = (torch.rand((m, n), generator=g, device="cuda", dtype=torch.float64) * 8 - 4).to(cb.dtype)
    c0 = cb[c_rows, c_cols].clone()
    alpha, beta = -1.0, 1.0
    tc.gemm_problem_device(gclass, bufs[0], bufs[1], bufs[2], ldw, m, n, k, lower=lower, exec_level=lvl,
                           alpha=alpha, beta=beta, **pos)
    torch.cuda.synchronize()
    c1 = cb[c_rows, c_cols]
    if lower:  # strict upper triangle untouched
        upper = torch.triu(torch.ones((m, n), dtype=torch.bool, device="cuda"), diagonal=1)
        assert torch.equal(c1[upper], c0[upper])
    rng = np.random.default_rng(k)
    ri, cj = _sample(48, m, rng), _sample(48, n, rng)
    ti, tj = torch.as_tensor(ri, device="cuda"), torch.as_tensor(cj, device="cuda")
    A = ob[a_rows, :k][ti].double().cpu().numpy()
    B = ob[b_rows, :k][tj].double().cpu().numpy()
    C0 = c0[ti][:, tj].double().cpu().numpy()
    got = c1[ti][:, tj].double().cpu().numpy()
    ref = np.asfortranarray(C0.copy())
    oracle.gemm_mixed(ref, np.asfortranarray(A), np.asfortranarray(B), alpha, beta, lvl)
    keep = (ri[:, None] >= cj[None, :]) if lower else np.ones_like(got, dtype=bool)
    got, ref, C0s = got[keep], ref[keep], C0[keep]
    assert np.all(np.isfinite(got))
    # the products summed in x87 extended precision (64-bit significand)
    LD = np.longdouble
    mag = ((np.abs(A).astype(LD) @ np.abs(B).T.astype(LD))[keep] * abs(alpha) + abs(beta) * np.abs(C0s))
    if lvl == 0:
        g32 = k * U32 / (1 - k * U32)
        ulp16 = np.spacing(np.maximum(np.abs(got), np.abs(ref)).astype(np.float16)).astype(LD)
        diff = np.abs(got.astype(LD) - ref.astype(LD))
        assert np.all(diff <= ulp16 + 2 * g32 * mag), float((diff / (ulp16 + 2 * g32 * mag)).max())
        d = np.abs(_half_order(got) - _half_order(ref))
        assert np.mean(d <= 1) >= 0.9, (int(d.max()), float(np.mean(d <= 1)))
        return
    exact = (LD(beta) * C0.astype(LD) + LD(alpha) * (A.astype(LD) @ B.T.astype(LD)))[keep]
    u = U64 if lvl == 2 else U32
    gamma = k * u / (1 - k * u)
    extra = 2.0 ** -19 if gclass in ("tc32", "mma32", "mma32w") else 0.0
    ulp = np.spacing(np.abs(exact).astype(np.float64 if lvl == 2 else np.float32)).astype(LD)
    e_gpu, e_or = np.abs(got.astype(LD) - exact), np.abs(ref.astype(LD) - exact)
    bound = (gamma + extra) * mag + ulp
    assert np.all(e_gpu <= bound), float((e_gpu / bound).max())
    assert np.all(e_or <= (gamma * mag + ulp)), "oracle outside its own bound"


@pytest.mark.gpu
@pytest.mark.parametrize("cls,m,n,k,ex,lower", [("tc16", 512, 512, 512, 0, 0), ("tc16", 1024, 768, 1024, 1, 0),
                                                ("tc16", 300, 200, 333, 0, 0), ("tc16", 512, 512, 2048, 1, 1),
                                                ("tc16", 2304, 1280, 640, 1, 0), ("tc16", 256, 256, 4096, 1, 1),
                                                ("tc32", 512, 512, 512, 1, 0), ("tc32", 300, 200, 333, 1, 0),
                                                ("tc32", 512, 512, 2048, 1, 1), ("tc32", 1024, 768, 1024, 1, 0)])
def test_cta_pair_gemm_bit_identical(tc, cls, m, n, k, ex, lower):
    """k_gemm_tc2 (tcgen05 cta_group::2, 256x256 tiles over a CTA pair; FP16
    kind and three-pass TF32) gives the single-CTA kernel's results bit for
    bit: the same K order per output element, only the tiling and the operand
    staging differ"""
    import torch

    def run(pair_min):
        tc.set_global_option("tc_pair_min_tiles", pair_min)
        g = torch.Generator(device="cuda").manual_seed(m + n + k)
        R = m + n
        ldw = ((k + n + 63) // 64) * 64
        b16 = (torch.rand((R, ldw), device="cuda", generator=g) * 2 - 1).half()
        b32 = torch.rand((R, ldw), device="cuda", generator=g) * 2 - 1
        tc.gemm_problem_device(cls, b16, b32, None, ldw, m, n, k, 0, 0, 0 if lower else m, 0, 0, k, ex, lower,
                               -1.0, 1.0)
        torch.cuda.synchronize()
        return (b16 if ex == 0 else b32)[:m, k:k + n].clone()

    try:
        single = run(0)
        pair = run(1)
    finally:
        tc.set_global_option("tc_pair_min_tiles", 512)
    assert torch.equal(single.view(torch.int16) if ex == 0 else single.view(torch.int32),
                       pair.view(torch.int16) if ex == 0 else pair.view(torch.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,ex,lower", [(512, 512, 512, 0, 0), (1024, 768, 1024, 1, 0), (300, 200, 333, 0, 0),
                                            (512, 512, 1024, 1, 1), (8192, 256, 512, 1, 0), (1000, 136, 200, 0, 0)])
def test_narrow_fp16_gemm_bit_identical(tc, m, n, k, ex, lower):
    """KIND_F16N (the FP16 kind on 128x128 tiles, option tc_narrow_max_tiles)
    gives the 128x256 kernel's results bit for bit"""
    import torch

    def run(narrow):
        tc.set_global_option("tc_narrow_max_tiles", 1 << 30 if narrow else 0)
        g = torch.Generator(device="cuda").manual_seed(m + n + k)
        ldw = ((k + n + 63) // 64) * 64
        b16 = (torch.rand((m + n, ldw), device="cuda", generator=g) * 2 - 1).half()
        b32 = torch.rand((m + n, ldw), device="cuda", generator=g) * 2 - 1
        tc.gemm_problem_device("tc16", b16, b32, None, ldw, m, n, k, 0, 0, 0 if lower else m, 0, 0, k, ex, lower,
                               -1.0, 1.0)
        torch.cuda.synchronize()
        return (b16 if ex == 0 else b32)[:m, k:k + n].clone()

    try:
        wide = run(False)
        narrow = run(True)
    finally:
        tc.set_global_option("tc_narrow_max_tiles", 0)
    assert torch.equal(wide.view(torch.int16) if ex == 0 else wide.view(torch.int32),
                       narrow.view(torch.int16) if ex == 0 else narrow.view(torch.int32))

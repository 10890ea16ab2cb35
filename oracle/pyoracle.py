"""ctypes face of the test oracles.  TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (the C restatement, ``oracle.c``) and, when it
was built here, ``oracle/_ref/libtreechol_ref.so`` (the compiled reference +
``ref_shim.cpp``).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline leg may import this module -- never the product package.

Matrices cross the boundary as Fortran-ordered float64 numpy arrays, i.e.
column-major exactly like the reference's TileView (matrix.hpp:11-24).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtreechol_ref.so")

HALF, SINGLE, DOUBLE = 0, 1, 2
STATUS = {0: "ok", 1: "not-positive-definite", 2: "numerical-breakdown",
          3: "singular-diagonal", 4: "invalid-argument"}
_NAMES = {"F16": HALF, "F32": SINGLE, "F64": DOUBLE}


def parse_levels(text: str) -> list[int]:
    """Minimal parser for the config strings the tests use (the full grammar
    lives in the product's PrecisionConfig::parse)."""
    t = text.strip().upper().replace("FP", "F")
    if t.startswith("PURE"):
        return [_NAMES[t[4:].strip()]]
    t = t.strip("[]")
    return [_NAMES[x.strip()] for x in t.split(",")]


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ivec(levels):
    arr = (C.c_int * len(levels))(*levels)
    return arr, len(levels)


@dataclass
class Flops:
    by_level: list = field(default_factory=lambda: [0, 0, 0])
    by_kernel: list = field(default_factory=lambda: [0, 0, 0, 0])
    calls: list = field(default_factory=lambda: [0, 0, 0, 0])

    @classmethod
    def from_array(cls, a):
        a = [int(x) for x in a]
        return cls(a[0:3], a[3:7], a[7:11])

    def total(self):
        return sum(self.by_level)

    def as_tuple(self):
        return tuple(self.by_level) + tuple(self.by_kernel) + tuple(self.calls)


class _Lib:
    def __init__(self, path, prefix):
        self.lib = C.CDLL(path)
        self.p = prefix

    def fn(self, name, res, *args):
        f = getattr(self.lib, self.p + name)
        f.restype = res
        f.argtypes = list(args)
        return f


class Oracle:
    """The C restatement (bit-exact to the reference; see test_oracle.py)."""

    def __init__(self, path=ORACLE_SO):
        L = _Lib(path, "or_")
        D, I, U64 = C.c_double, C.c_int, C.c_uint64
        PD, PI = C.POINTER(C.c_double), C.POINTER(C.c_int)
        PU = C.POINTER(C.c_uint64)
        self._round = L.fn("round_to", D, D, I)
        self._gen = L.fn("spd_generate", None, I, U64, PD)
        self._err = L.fn("factorization_error", D, I, PD, I, PD, I)
        self._fb = L.fn("flop_breakdown", None, I, I, PI, I, PU)
        self._potrf = L.fn("tree_potrf", I, I, PD, I, I, PI, I, I, PU, C.c_char_p, I)
        self._potrs = L.fn("potrs", None, I, PD, I, PD, I, I)
        self._gemm = L.fn("gemm_mixed", None, PD, I, I, I, PD, I, I, PD, I, D, D, I, PU)
        self._trsm = L.fn("trsm_leaf", I, PD, I, I, I, PD, I, I, I, PU, PI)
        self._syrk = L.fn("syrk_leaf", None, PD, I, I, PD, I, I, D, D, I, PU)
        self._potrf_leaf = L.fn("potrf_leaf", I, PD, I, I, I, I, PU, PI)
        self._set_threads = L.fn("set_threads", None, I)
        self._get_threads = L.fn("get_threads", I)

    def set_threads(self, t):
        self._set_threads(int(t))

    def threads(self):
        return self._get_threads()

    def round_to(self, x, p):
        return self._round(float(x), int(p))

    def spd_generate(self, n, seed):
        a = np.empty((n, n), dtype=np.float64, order="F")
        self._gen(n, seed, _dptr(a))
        return a

    def factorization_error(self, a, l):
        n = a.shape[0]
        return self._err(n, _dptr(a), n, _dptr(l), n)

    def flop_breakdown(self, n, b, levels):
        out = (C.c_uint64 * 11)()
        lv, nl = _ivec(levels)
        self._fb(n, b, lv, nl, out)
        return Flops.from_array(out)

    def tree_potrf(self, a, b, levels, quantize=True):
        """In place on a (Fortran float64); returns (status, detail, Flops)."""
        assert a.flags.f_contiguous and a.dtype == np.float64
        n = a.shape[0]
        out = (C.c_uint64 * 11)()
        lv, nl = _ivec(levels)
        buf = C.create_string_buffer(512)
        st = self._potrf(n, _dptr(a), n, b, lv, nl, int(bool(quantize)), out, buf, 512)
        return STATUS[st], buf.value.decode(), Flops.from_array(out)

    def factor(self, a, b, levels, quantize=True):
        """factor_matrix: returns (status, detail, L, rel_error, Flops)."""
        l = np.array(a, dtype=np.float64, order="F", copy=True)
        st, det, fl = self.tree_potrf(l, b, levels, quantize)
        rel = self.factorization_error(a, l) if st == "ok" else float("nan")
        return st, det, l, rel, fl

    def potrs(self, l, rhs):
        n = l.shape[0]
        x = np.array(rhs, dtype=np.float64, order="F", copy=True)
        if x.ndim == 1:
            x = x.reshape(n, 1, order="F")
        self._potrs(n, _dptr(l), n, _dptr(x), n, x.shape[1])
        return x

    def gemm_mixed(self, c, a, b, alpha, beta, level):
        m, n = c.shape
        k = a.shape[1]
        self._gemm(_dptr(c), m, n, m, _dptr(a), k, m, _dptr(b), n, alpha, beta, level, None)

    def syrk_leaf(self, c, a, alpha, beta, level):
        n = c.shape[0]
        self._syrk(_dptr(c), n, n, _dptr(a), a.shape[1], n, alpha, beta, level, None)

    def trsm_leaf(self, b, l, level):
        m, n = b.shape
        idx = C.c_int(0)
        st = self._trsm(_dptr(b), m, n, m, _dptr(l), n, 0, level, None, C.byref(idx))
        return STATUS[st], idx.value

    def potrf_leaf(self, a, level):
        n = a.shape[0]
        idx = C.c_int(0)
        st = self._potrf_leaf(_dptr(a), n, n, 0, level, None, C.byref(idx))
        return STATUS[st], idx.value


class Reference:
    """The compiled reference (only where oracle/_ref was built)."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self, path=REF_SO):
        L = _Lib(path, "ref_")
        D, I, U64 = C.c_double, C.c_int, C.c_uint64
        PD, PI, PU = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_uint64)
        self._round = L.fn("round_to", D, D, I)
        self._gen = L.fn("spd_generate", None, I, U64, PD)
        self._err = L.fn("factorization_error", D, I, PD, PD)
        self._fb = L.fn("flop_breakdown", None, I, I, PI, I, PU)
        self._potrf = L.fn("tree_potrf", I, I, PD, I, I, PI, I, I, PU, C.c_char_p, I)
        self._time = L.fn("time_factor", D, I, PD, I, PI, I, I)
        self._gemm = L.fn("gemm_mixed", None, PD, I, I, I, PD, I, I, PD, I, D, D, I)
        self._trsm = L.fn("trsm_leaf", I, PD, I, I, I, PD, I, I)
        self._syrk = L.fn("syrk_leaf", None, PD, I, I, PD, I, I, D, D, I)
        self._potrf_leaf = L.fn("potrf_leaf", I, PD, I, I, I)

    def round_to(self, x, p):
        return self._round(float(x), int(p))

    def spd_generate(self, n, seed):
        a = np.empty((n, n), dtype=np.float64, order="F")
        self._gen(n, seed, _dptr(a))
        return a

    def factorization_error(self, a, l):
        return self._err(a.shape[0], _dptr(a), _dptr(l))

    def flop_breakdown(self, n, b, levels):
        out = (C.c_uint64 * 11)()
        lv, nl = _ivec(levels)
        self._fb(n, b, lv, nl, out)
        return Flops.from_array(out)

    def tree_potrf(self, a, b, levels, quantize=True):
        n = a.shape[0]
        out = (C.c_uint64 * 11)()
        lv, nl = _ivec(levels)
        buf = C.create_string_buffer(512)
        st = self._potrf(n, _dptr(a), n, b, lv, nl, int(bool(quantize)), out, buf, 512)
        return STATUS[st], buf.value.decode(), Flops.from_array(out)

    def time_factor_ms(self, a, b, levels, quantize=True):
        lv, nl = _ivec(levels)
        return self._time(a.shape[0], _dptr(a), b, lv, nl, int(bool(quantize)))

    def gemm_mixed(self, c, a, b, alpha, beta, level):
        m, n = c.shape
        self._gemm(_dptr(c), m, n, m, _dptr(a), a.shape[1], m, _dptr(b), n, alpha, beta, level)

    def syrk_leaf(self, c, a, alpha, beta, level):
        n = c.shape[0]
        self._syrk(_dptr(c), n, n, _dptr(a), a.shape[1], n, alpha, beta, level)

    def trsm_leaf(self, b, l, level):
        m, n = b.shape
        return STATUS[self._trsm(_dptr(b), m, n, m, _dptr(l), n, level)]

    def potrf_leaf(self, a, level):
        n = a.shape[0]
        return STATUS[self._potrf_leaf(_dptr(a), n, n, level)]

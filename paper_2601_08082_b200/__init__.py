"""treechol-b200: B200-native nested recursive mixed-precision Cholesky.

Python host mirror of the reference's public interface
(/root/reference/proj/include/treechol/*.hpp) over the C ABI of
``libtreechol_b200.so`` (include/treechol_c.h).  Names, argument meaning and
error behaviour follow the reference:

    PrecisionConfig.parse / to_string / at_depth / leaf   precision.hpp:81-99
    flop_breakdown(n, b, config)                          analysis.hpp:44
    factor_matrix(a, config, b, quantize) -> FactorReport analysis.hpp:48
    spd_generate(n, seed), factorization_error(a, l)      analysis.hpp:33-38
    NotPositiveDefinite / NumericalBreakdown / ...        errors.hpp:8-62

plus the device API the reference does not have: ``Plan`` (build once, factor
device-resident matrices through a cached CUDA graph), ``potrs`` and the
GPU backward-error metrics.  There is no CPU fallback: every compute call
needs a CUDA device and raises ``NoDevice`` without one.

Matrices are column-major doubles exactly like the reference's TileView.  On
the host that is a Fortran-ordered numpy array; on the device a torch tensor
``t`` of shape (n, n) whose memory is column-major, i.e. ``t[j, i] = A(i, j)``
(``to_device`` / ``from_device`` convert).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtreechol_b200.so")

HALF, SINGLE, DOUBLE = 0, 1, 2
_LEVEL_NAMES = ("F16", "F32", "F64")
POTRF, TRSM, SYRK, GEMM = 0, 1, 2, 3
KERNEL_NAMES = ("POTRF-leaf", "TRSM-leaf", "SYRK-leaf", "GEMM")  # flops.cpp:5-12

TC_OK, TC_NPD, TC_BREAKDOWN, TC_SINGULAR, TC_INVALID, TC_SYNTAX, TC_VALIDATION, TC_CUDA, TC_NO_DEVICE = range(9)

OP_TYPES = ("import", "export", "check", "quant", "dequant", "shadow", "potrf", "trsm", "gemm", "inverse")
GEMM_CLASSES = ("tc16", "simt_f16", "simt_f32", "simt_f16d", "simt_f32d", "simt_f64", "tc32", "mma32", "mma32w")


# ---------------------------------------------------------------- errors.hpp
class Error(RuntimeError):
    """treechol::Error"""


class SyntaxError_(Error):
    """treechol::SyntaxError (config grammar)"""


class ValidationError(Error):
    """treechol::ValidationError (non-monotone config)"""


class InvalidArgument(Error):
    """treechol::InvalidArgument"""


class NotPositiveDefinite(Error):
    def __init__(self, index: int, msg: str = ""):
        super().__init__(msg or f"matrix is not positive definite: pivot {index} is non-positive or non-finite")
        self.index = index


class SingularDiagonal(Error):
    def __init__(self, index: int, msg: str = ""):
        super().__init__(msg or f"singular triangular factor: diagonal entry {index} is zero or non-finite")
        self.index = index


class NumericalBreakdown(Error):
    """treechol::NumericalBreakdown"""


class CudaError(Error):
    """device / runtime failure (no reference counterpart)"""


class NoDevice(Error):
    """no CUDA device: the library has no CPU path"""


# ---------------------------------------------------------------- C structs
class _Flops(C.Structure):
    _fields_ = [("by_level", C.c_uint64 * 3), ("by_kernel", C.c_uint64 * 4), ("calls", C.c_uint64 * 4)]


class _Info(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("status", "index", "row0", "row1", "col0", "col1", "elem_row", "elem_col", "diagonal")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2601_08082_b200/csrc)")
    lib = C.CDLL(LIB_PATH)
    I, D, P, U64 = C.c_int, C.c_double, C.c_void_p, C.c_uint64
    PI = C.POINTER(C.c_int)
    sig = {
        "tc_config_parse": (I, [C.c_char_p, PI, PI]),
        "tc_config_to_string": (I, [PI, I, C.c_char_p, I]),
        "tc_flop_breakdown": (I, [I, I, PI, I, C.POINTER(_Flops)]),
        "tc_plan_create": (I, [I, I, PI, I, I, I, C.POINTER(P)]),
        "tc_plan_destroy": (None, [P]),
        "tc_plan_flops": (I, [P, C.POINTER(_Flops)]),
        "tc_plan_run_flops": (I, [P, C.POINTER(_Flops)]),
        "tc_plan_stats": (I, [P, PI, PI, PI]),
        "tc_plan_set_option": (I, [P, C.c_char_p, I]),
        "tc_plan_op_info": (I, [P, I, PI, PI, PI, C.POINTER(D), PI]),
        "tc_plan_op_deps": (I, [P, I, PI, I]),
        "tc_potrf_device": (I, [P, P, I, P, I, P, C.POINTER(_Info)]),
        "tc_potrf_host": (I, [P, P, I, C.POINTER(_Info)]),
        "tc_plan_profile": (I, [P, P, I, P, I, P, C.POINTER(C.c_float), I]),
        "tc_plan_status": (I, [P, C.POINTER(_Info)]),
        "tc_plan_op_probs": (I, [P, I, C.POINTER(C.c_int), I]),
        "tc_plan_timeline": (I, [P, P, I, P, I, P, C.POINTER(C.c_float), C.POINTER(C.c_float), I]),
        "tc_plan_trace_device": (I, [P, P, I, P, I, P, C.POINTER(C.c_float), I]),
        "tc_plan_trace_host": (I, [P, P, I, P, C.POINTER(C.c_float), I, C.POINTER(C.c_float), I,
                                   C.POINTER(C.c_float), I]),
        "tc_plan_timeline_host": (I, [P, P, I, P, C.POINTER(C.c_float), C.POINTER(C.c_float), I,
                                      C.POINTER(C.c_float), I, C.POINTER(C.c_float), I]),
        "tc_info_message": (I, [P, C.POINTER(_Info), C.c_char_p, I]),
        "tc_potrs_device": (I, [I, P, I, P, I, I, P]),
        "tc_potrs_batch_device": (I, [I, I, C.POINTER(P), I, C.POINTER(P), I, I, P]),
        "tc_spd_generate_host": (I, [I, U64, P, I]),
        "tc_spd_generate_device": (I, [I, U64, P, I, P]),
        "tc_factorization_error_device": (I, [I, P, I, P, I, C.POINTER(D), P]),
        "tc_solve_residual_device": (I, [I, P, I, P, P, C.POINTER(D), P]),
        "tc_debug_gemm": (I, [I, I, I, I, I, D, I, I, C.POINTER(C.c_float)]),
        "tc_gemm_problem_device": (I, [I, P, P, P, C.c_longlong, PI, D, D, P]),
        "tc_set_global_option": (I, [C.c_char_p, I]),
        "tc_debug_gemm_stamps": (I, [C.POINTER(C.c_uint64)]),
        "tc_debug_fp64_probe": (D, [I, I, I]),
        "tc_debug_mma_probe": (D, [I, I]),
        "tc_plan_create_trsm": (I, [I, I, I, PI, I, I, C.POINTER(P)]),
        "tc_plan_create_syrk_rows": (I, [I, I, I, PI, I, I, I, C.POINTER(P)]),
        "tc_plan_set_external_absmax": (I, [P, D]),
        "tc_plan_create_trsm_ext": (I, [I, I, I, PI, I, I, C.POINTER(P)]),
        "tc_plan_create_syrk_rows_ext": (I, [I, I, I, PI, I, I, I, C.POINTER(P)]),
        "tc_plan_input_rows": (I, [P, PI, PI]),
        "tc_plan_device_bytes": (I, [P, C.POINTER(C.c_ulonglong)]),
        "tc_plan_level_buffer": (I, [P, I, C.POINTER(P), C.POINTER(C.c_longlong), PI, PI]),
        "tc_level_image_device": (I, [I, I, P, I, I, I, P, C.c_longlong, P]),
        "tc_plan_extent": (I, [P, PI, PI]),
        "tc_absmax_device": (I, [I, I, P, I, C.POINTER(D), P]),
        "tc_batch_create": (I, [I, I, PI, I, I, I, C.POINTER(P)]),
        "tc_batch_destroy": (None, [P]),
        "tc_batch_set_option": (I, [P, C.c_char_p, I]),
        "tc_batch_run": (I, [P, I, C.POINTER(P), I, C.POINTER(P), I, I, PI, PI]),
        "tc_batch_solve_ms": (I, [P, C.POINTER(C.c_float)]),
        "tc_round_host": (I, [I, I, P, I, I, I]),
        "tc_quantize_host": (I, [I, I, P, I, I, C.POINTER(D)]),
        "tc_dequantize_host": (I, [I, I, P, I, I, D]),
        "tc_potrf_leaf_host": (I, [I, P, I, I, I, PI]),
        "tc_trsm_leaf_host": (I, [I, I, P, I, P, I, I, I, PI]),
        "tc_gemm_mixed_host": (I, [I, I, I, P, I, P, I, P, I, D, D, I, I, I]),
        "tc_last_error": (C.c_char_p, []),
        "tc_device_available": (I, []),
        "tc_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = tuple(n for n in dir(_lib) if n.startswith("tc_"))


def lib():
    return _lib


def _last_error() -> str:
    return (_lib.tc_last_error() or b"").decode()


def _raise(code: int, info: _Info | None = None):
    msg = _last_error()
    if code == TC_OK:
        return
    if code == TC_NPD:
        raise NotPositiveDefinite(info.index if info else -1, msg)
    if code == TC_SINGULAR:
        raise SingularDiagonal(info.index if info else -1, msg)
    if code == TC_BREAKDOWN:
        raise NumericalBreakdown(msg)
    if code == TC_SYNTAX:
        raise SyntaxError_(msg)
    if code == TC_VALIDATION:
        raise ValidationError(msg)
    if code == TC_INVALID:
        raise InvalidArgument(msg)
    if code == TC_NO_DEVICE:
        raise NoDevice(msg)
    raise CudaError(msg)


def version() -> str:
    return _lib.tc_version().decode()


def device_available() -> bool:
    return bool(_lib.tc_device_available())


# ---------------------------------------------------------------- precision.hpp
class Precision:
    Half, Single, Double = HALF, SINGLE, DOUBLE


def range_max(p: int) -> float:  # precision.hpp:20-26
    return (65504.0, 3.4028234663852886e38, 1.7976931348623157e308)[p]


def unit_roundoff(p: int) -> float:  # precision.hpp:28-34
    return (2.0 ** -11, 2.0 ** -24, 2.0 ** -53)[p]


def precision_name(p: int) -> str:
    return _LEVEL_NAMES[p]


@dataclass(frozen=True)
class PrecisionConfig:
    """precision.hpp:81-99: outer -> inner levels, saturating at the last."""
    levels: tuple

    def at_depth(self, d: int) -> int:
        return self.levels[min(d, len(self.levels) - 1)]

    def leaf(self) -> int:
        return self.levels[-1]

    def to_string(self) -> str:
        arr = (C.c_int * len(self.levels))(*self.levels)
        buf = C.create_string_buffer(128)
        _raise(_lib.tc_config_to_string(arr, len(self.levels), buf, 128))
        return buf.value.decode()

    def __str__(self):
        return self.to_string()

    @staticmethod
    def parse(text: str) -> "PrecisionConfig":
        arr = (C.c_int * 16)()
        n = C.c_int(0)
        _raise(_lib.tc_config_parse(text.encode(), arr, C.byref(n)))
        return PrecisionConfig(tuple(arr[i] for i in range(n.value)))


def _cfg(config) -> PrecisionConfig:
    if isinstance(config, PrecisionConfig):
        return config
    if isinstance(config, str):
        return PrecisionConfig.parse(config)
    return PrecisionConfig(tuple(int(x) for x in config))


# ---------------------------------------------------------------- flops.hpp
@dataclass
class FlopBreakdown:
    by_level: list = field(default_factory=lambda: [0, 0, 0])
    by_kernel: list = field(default_factory=lambda: [0, 0, 0, 0])
    calls: list = field(default_factory=lambda: [0, 0, 0, 0])

    @classmethod
    def _from(cls, f: _Flops):
        return cls(list(f.by_level), list(f.by_kernel), list(f.calls))

    def total(self) -> int:
        return sum(self.by_level)

    def level_fraction(self, p: int) -> float:
        t = self.total()
        return 0.0 if t == 0 else self.by_level[p] / t

    def kernel_fraction(self, k: int) -> float:
        t = self.total()
        return 0.0 if t == 0 else self.by_kernel[k] / t

    def as_tuple(self):
        return tuple(self.by_level) + tuple(self.by_kernel) + tuple(self.calls)


def flop_breakdown(n: int, b: int, config) -> FlopBreakdown:
    """analysis.cpp:64-120 (static, no device)."""
    cfg = _cfg(config)
    arr = (C.c_int * len(cfg.levels))(*cfg.levels)
    out = _Flops()
    _raise(_lib.tc_flop_breakdown(n, b, arr, len(cfg.levels), C.byref(out)))
    return FlopBreakdown._from(out)


def potrf_flops(n: int) -> int:
    """n(n+1)(2n+1)/6, the total of every tree (analysis.cpp:66-68)."""
    return n * (n + 1) * (2 * n + 1) // 6


# ---------------------------------------------------------------- device glue
def _ptr(t) -> int:
    """raw device / host pointer of a torch tensor or numpy array"""
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def _stream_ptr(stream):
    if stream is None:
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def to_device(a: np.ndarray, device="cuda"):
    """Fortran float64 (n, m) -> torch tensor with the same column-major memory."""
    import torch
    a = np.asfortranarray(a, dtype=np.float64)
    return torch.from_numpy(a.T).to(device)


def from_device(t) -> np.ndarray:
    """inverse of to_device: a Fortran-ordered numpy array"""
    return np.asfortranarray(t.detach().cpu().numpy().T)


class _DevView:
    """__cuda_array_interface__ over raw device memory owned elsewhere"""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def level_image_device(src, m: int, n: int, level: int, dst, ldd: int, lower: bool = True, stream=None):
    """dst (row-major, ld ldd) = rn_level of the m x n column-major double
    block src (torch tensor (n, lds)), strict upper triangle zeroed when
    lower (tc_level_image_device)"""
    lds = src.shape[1] if src.dim() == 2 else m
    _raise(_lib.tc_level_image_device(m, n, _ptr(src), lds, int(level), int(bool(lower)), _ptr(dst), int(ldd),
                                      _stream_ptr(stream)))


def _check_dev(t, n, what, cols=None):
    """a contiguous CUDA float64 column-major tensor (cols', ld) with
    ld >= n rows and cols' >= cols (default n) columns; returns ld"""
    import torch
    cols = n if cols is None else cols
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise InvalidArgument(f"{what} must be a CUDA float64 tensor")
    if t.dim() != 2 or t.shape[1] < n or t.shape[0] < cols or not t.is_contiguous():
        raise InvalidArgument(f"{what} must be a contiguous ({cols}+ columns, ld >= {n}) tensor, "
                              f"got shape {tuple(t.shape)}")
    return t.shape[1]


@dataclass
class FactorStatus:
    status: str            # ok | not-positive-definite | numerical-breakdown | singular-diagonal
    detail: str = ""
    index: int = -1
    info: _Info | None = None


_STATUS_NAMES = {TC_OK: "ok", TC_NPD: "not-positive-definite", TC_BREAKDOWN: "numerical-breakdown",
                 TC_SINGULAR: "singular-diagonal"}


class Plan:
    """build_tree + tree_potrf for one (n, b, config, quantize), planned once
    (tree.hpp:42-66).  Device workspace is allocated on the first factor."""

    def __init__(self, n: int, b: int, config, quantize: bool = True, leaf_size: int = 0, use_tc: bool = True,
                 use_graph: bool = True, n_streams: int = 0, use_tc32: bool = True):
        self.cfg = _cfg(config)
        self.n, self.b, self.quantize = int(n), int(b), bool(quantize)
        arr = (C.c_int * len(self.cfg.levels))(*self.cfg.levels)
        h = C.c_void_p()
        _raise(_lib.tc_plan_create(self.n, self.b, arr, len(self.cfg.levels), int(self.quantize), int(leaf_size),
                                   C.byref(h)))
        self._h = h
        self._extent()
        if not use_tc:
            self.set_option("use_tc", 0)
        if not use_tc32:
            self.set_option("use_tc32", 0)
        if not use_graph:
            self.set_option("use_graph", 0)
        if n_streams:
            self.set_option("n_streams", n_streams)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.tc_plan_destroy(h)
            self._h = None

    @classmethod
    def _wrap(cls, h, n, b, config, rows):
        self = cls.__new__(cls)
        self.cfg = _cfg(config)
        self.n, self.b, self.quantize = int(rows), int(b), True
        self._h = h
        self._extent()
        return self

    def _extent(self):
        """rows x cols of the column-major operand the plan reads and writes
        (tc_plan_extent / tc_plan_input_rows; n x n for a whole
        factorization; the compact distributed pieces take only their rows)"""
        r, c = C.c_int(), C.c_int()
        _raise(_lib.tc_plan_extent(self._h, C.byref(r), C.byref(c)))
        r0, nr = C.c_int(), C.c_int()
        _raise(_lib.tc_plan_input_rows(self._h, C.byref(r0), C.byref(nr)))
        self.row0, self.rows, self.cols = r0.value, nr.value, c.value

    def device_bytes(self) -> int:
        """device workspace of the plan (level-buffer windows, leaf inverses)"""
        out = C.c_ulonglong()
        _raise(_lib.tc_plan_device_bytes(self._h, C.byref(out)))
        return out.value

    def level_buffer(self, level: int):
        """(tensor, row_lo): the allocated window of a level buffer as a torch
        tensor view (rows x ld, row-major) whose row 0 is buffer row row_lo;
        valid while the plan lives"""
        import torch
        ptr, ld, lo, hi = C.c_void_p(), C.c_longlong(), C.c_int(), C.c_int()
        _raise(_lib.tc_plan_level_buffer(self._h, int(level), C.byref(ptr), C.byref(ld), C.byref(lo), C.byref(hi)))
        typestr = ("<f2", "<f4", "<f8")[level]
        view = _DevView(ptr.value, (hi.value - lo.value, ld.value), typestr)
        t = torch.as_tensor(view, device="cuda")
        t._tc_owner = self  # keep the plan (and its workspace) alive
        return t, lo.value

    @classmethod
    def panel_trsm(cls, n1: int, m: int, b: int, config, leaf_size: int = 0) -> "Plan":
        """distributed C5 piece: rows [0, n1) = factored L11, rows [n1, n1+m)
        = a row block of A21 to quantize (external alpha) and solve
        (tc_plan_create_trsm)"""
        cfg = _cfg(config)
        arr = (C.c_int * len(cfg.levels))(*cfg.levels)
        h = C.c_void_p()
        _raise(_lib.tc_plan_create_trsm(n1, m, b, arr, len(cfg.levels), leaf_size, C.byref(h)))
        return cls._wrap(h, n1, b, cfg, n1 + m)

    @classmethod
    def panel_trsm_ext(cls, n1: int, m: int, b: int, config, leaf_size: int = 0) -> "Plan":
        """compact distributed TRSM piece (tc_plan_create_trsm_ext): the
        caller writes rn_p(L11) into level buffer p rows [0, n1); the
        operand is only the m panel rows (tensor (n1, m))"""
        cfg = _cfg(config)
        arr = (C.c_int * len(cfg.levels))(*cfg.levels)
        h = C.c_void_p()
        _raise(_lib.tc_plan_create_trsm_ext(n1, m, b, arr, len(cfg.levels), leaf_size, C.byref(h)))
        return cls._wrap(h, n1, b, cfg, n1 + m)

    @classmethod
    def panel_syrk_rows_ext(cls, n2: int, k: int, b: int, config, row_lo: int, row_hi: int) -> "Plan":
        """compact distributed SYRK piece (tc_plan_create_syrk_rows_ext): the
        caller writes the solved panel's level image into level buffer p rows
        [row_hi, row_hi + n2); the operand is A22's rows [row_lo, row_hi)
        only (tensor (n2, row_hi - row_lo))"""
        cfg = _cfg(config)
        arr = (C.c_int * len(cfg.levels))(*cfg.levels)
        h = C.c_void_p()
        _raise(_lib.tc_plan_create_syrk_rows_ext(n2, k, b, arr, len(cfg.levels), row_lo, row_hi, C.byref(h)))
        return cls._wrap(h, n2, b, cfg, row_hi + n2)

    @classmethod
    def panel_syrk_rows(cls, n2: int, k: int, b: int, config, row_lo: int, row_hi: int) -> "Plan":
        """distributed C5 piece: rows [0, n2) = A22, rows [n2, 2 n2) = the
        solved A21; tree_syrk on A22's rows [row_lo, row_hi)
        (tc_plan_create_syrk_rows)"""
        cfg = _cfg(config)
        arr = (C.c_int * len(cfg.levels))(*cfg.levels)
        h = C.c_void_p()
        _raise(_lib.tc_plan_create_syrk_rows(n2, k, b, arr, len(cfg.levels), row_lo, row_hi, C.byref(h)))
        return cls._wrap(h, n2, b, cfg, 2 * n2)

    def set_external_absmax(self, amax: float):
        _raise(_lib.tc_plan_set_external_absmax(self._h, float(amax)))

    def set_option(self, key: str, value: int):
        _raise(_lib.tc_plan_set_option(self._h, key.encode(), int(value)))

    def flops(self) -> FlopBreakdown:
        out = _Flops()
        _raise(_lib.tc_plan_flops(self._h, C.byref(out)))
        return FlopBreakdown._from(out)

    def run_flops(self) -> FlopBreakdown:
        out = _Flops()
        _raise(_lib.tc_plan_run_flops(self._h, C.byref(out)))
        return FlopBreakdown._from(out)

    def stats(self):
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        _raise(_lib.tc_plan_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"ops": a.value, "launches": b.value, "gemm_problems": c.value}

    def op_info(self, i: int):
        t, g, lv = C.c_int(), C.c_int(), C.c_int()
        fl = C.c_double()
        r = (C.c_int * 4)()
        _raise(_lib.tc_plan_op_info(self._h, i, C.byref(t), C.byref(g), C.byref(lv), C.byref(fl), r))
        return {"type": OP_TYPES[t.value], "gclass": GEMM_CLASSES[g.value] if g.value >= 0 else None,
                "level": lv.value, "flops": fl.value, "rect": tuple(r)}

    def op_probs(self, i: int):
        """GEMM problems of op i: dicts of m, n, k, a_r0, a_c0, a_kwrap, b_buf,
        b_r0, b_c0, c_r0, c_c0, exec_level, lower"""
        keys = ("m", "n", "k", "a_r0", "a_c0", "a_kwrap", "b_buf", "b_r0", "b_c0", "c_r0", "c_c0", "exec_level",
                "lower")
        cnt = _lib.tc_plan_op_probs(self._h, i, None, 0)
        if cnt < 0:
            _raise(cnt)
        arr = (C.c_int * (13 * max(cnt, 1)))()
        _lib.tc_plan_op_probs(self._h, i, arr, cnt)
        return [dict(zip(keys, arr[13 * q:13 * q + 13])) for q in range(cnt)]

    def op_deps(self, i: int):
        cap = 64
        while True:
            arr = (C.c_int * cap)()
            k = _lib.tc_plan_op_deps(self._h, i, arr, cap)
            if k < 0:
                raise InvalidArgument("bad op index")
            if k <= cap:
                return list(arr[:k])
            cap = k

    def _status(self, code: int, info: _Info) -> FactorStatus:
        if code in (TC_OK, TC_NPD, TC_BREAKDOWN, TC_SINGULAR):
            buf = C.create_string_buffer(512)
            _lib.tc_info_message(self._h, C.byref(info), buf, 512)
            return FactorStatus(_STATUS_NAMES[code], buf.value.decode(), info.index, info)
        _raise(code, info)

    def factor_device(self, a_in, l_out=None, stream=None, sync: bool = True):
        """Device-resident tree_potrf: reads a_in, writes L's lower triangle
        into l_out (default: in place).  Returns FactorStatus when sync."""
        n, cols = self.rows, self.cols
        lda = _check_dev(a_in, n, "a_in", cols)
        l_out = a_in if l_out is None else l_out
        ldl = _check_dev(l_out, n, "l_out", cols)
        info = _Info()
        code = _lib.tc_potrf_device(self._h, _ptr(a_in), lda, _ptr(l_out), ldl, _stream_ptr(stream),
                                    C.byref(info) if sync else None)
        if not sync:
            _raise(code)
            return None
        return self._status(code, info)

    def status(self) -> FactorStatus:
        info = _Info()
        code = _lib.tc_plan_status(self._h, C.byref(info))
        return self._status(code, info)

    def factor_host(self, a: np.ndarray) -> FactorStatus:
        """tree_potrf on a host Fortran float64 array, in place (TileView contract)."""
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.f_contiguous):
            raise InvalidArgument("a must be a Fortran-ordered float64 array")
        if a.ndim != 2 or a.shape[0] < self.rows or a.shape[1] < self.cols:
            raise InvalidArgument(f"a must be at least {self.rows} x {self.cols}, got {a.shape}")
        info = _Info()
        code = _lib.tc_potrf_host(self._h, a.ctypes.data, a.shape[0], C.byref(info))
        return self._status(code, info)

    def timeline(self, a_in, l_out, stream=None):
        """eager multi-stream run; per-op (start, end) ms from the start"""
        n_ops = self.stats()["ops"]
        t0, t1 = (C.c_float * n_ops)(), (C.c_float * n_ops)()
        _raise(_lib.tc_plan_timeline(self._h, _ptr(a_in), _check_dev(a_in, self.rows, "a_in", self.cols),
                                     _ptr(l_out), _check_dev(l_out, self.rows, "l_out", self.cols),
                                     _stream_ptr(stream), t0, t1, n_ops))
        return list(t0), list(t1)

    def trace(self, a_in, l_out, stream=None):
        """development: one run of the DAG graph with a timer stamp after
        every op; per-op completion ms from the graph's root"""
        n_ops = self.stats()["ops"]
        out = (C.c_float * n_ops)()
        _raise(_lib.tc_plan_trace_device(self._h, _ptr(a_in), _check_dev(a_in, self.rows, "a_in", self.cols),
                                         _ptr(l_out), _check_dev(l_out, self.rows, "l_out", self.cols),
                                         _stream_ptr(stream), out, n_ops))
        return list(out)

    def profile(self, a_in, l_out, stream=None):
        """serialized eager run; per-op device milliseconds"""
        n_ops = self.stats()["ops"]
        out = (C.c_float * n_ops)()
        _raise(_lib.tc_plan_profile(self._h, _ptr(a_in), _check_dev(a_in, self.rows, "a_in", self.cols),
                                    _ptr(l_out), _check_dev(l_out, self.rows, "l_out", self.cols),
                                    _stream_ptr(stream), out, n_ops))
        return list(out)


class Batch:
    """Batched tree_potrf + POTRS of independent systems on one device
    (tc_batch_*; BASELINE config C4).  `concurrency` plans run side by side."""

    def __init__(self, n: int, b: int, config, quantize: bool = True, concurrency: int = 4):
        self.cfg = _cfg(config)
        self.n = int(n)
        arr = (C.c_int * len(self.cfg.levels))(*self.cfg.levels)
        h = C.c_void_p()
        _raise(_lib.tc_batch_create(self.n, int(b), arr, len(self.cfg.levels), int(bool(quantize)), int(concurrency),
                                    C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.tc_batch_destroy(h)
            self._h = None

    def set_option(self, key: str, value: int):
        _raise(_lib.tc_batch_set_option(self._h, key.encode(), int(value)))

    def run(self, a_list, b_list=None):
        """factor every a_list[k] in place (device column-major tensors, see
        to_device) and solve with b_list[k] (device tensors (nrhs, n)) if
        given; returns the per-system status names"""
        import torch
        k = len(a_list)
        lda = _check_dev(a_list[0], self.n, "A[0]") if k else self.n
        for i, a in enumerate(a_list):  # one leading dimension for the whole batch
            if _check_dev(a, self.n, f"A[{i}]") != lda or a.shape != a_list[0].shape:
                raise InvalidArgument(f"A[{i}] must have the shape of A[0] {tuple(a_list[0].shape)}")
        pa = (C.c_void_p * k)(*[_ptr(a) for a in a_list])
        pb, ldb, nrhs = None, self.n, 1
        if b_list is not None:  # entries may be None: that system is factored only
            if len(b_list) != k:
                raise InvalidArgument("b_list must have one entry (or None) per system")
            b2 = []
            for i, x in enumerate(b_list):
                if x is not None:
                    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64
                            and x.is_contiguous() and x.dim() in (1, 2)):
                        raise InvalidArgument(f"B[{i}] must be a contiguous CUDA float64 tensor (nrhs, ldb)")
                    x = x if x.dim() == 2 else x.view(1, -1)
                b2.append(x)
            first = next((x for x in b2 if x is not None), None)
            if first is not None:
                ldb, nrhs = first.shape[1], first.shape[0]
                if ldb < self.n:
                    raise InvalidArgument(f"B rows ({ldb}) < n ({self.n})")
                for i, x in enumerate(b2):
                    if x is not None and x.shape != first.shape:
                        raise InvalidArgument(f"B[{i}] must have the shape of the first B {tuple(first.shape)}")
            pb = (C.c_void_p * k)(*[None if x is None else _ptr(x) for x in b2])
        st = (C.c_int * max(k, 1))()
        idx = (C.c_int * max(k, 1))()
        code = _lib.tc_batch_run(self._h, k, pa, lda, pb, ldb, nrhs, st, idx)
        if code not in (TC_OK, TC_NPD, TC_BREAKDOWN, TC_SINGULAR):
            _raise(code)
        return [_STATUS_NAMES[st[i]] for i in range(k)]

    def last_solve_ms(self) -> float:
        """device ms of the last run's batched solve phase (0 if none)"""
        ms = C.c_float()
        _raise(_lib.tc_batch_solve_ms(self._h, C.byref(ms)))
        return ms.value


# ---------------------------------------------------------------- kernels.hpp / tree.hpp block ops
# The reference's kernel-level API on host Fortran float64 arrays, executed
# on the device in the reference's scalar operation order (k_blockops.cu).

def _fortran(x, what):
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.f_contiguous):
        raise InvalidArgument(f"{what} must be a Fortran-ordered float64 array")
    return x


def round_matrix(tile: np.ndarray, level: int, lower: bool = False):
    """kernels.cpp:9-16 (round_lower of tree.cpp:33-40 with lower=True)"""
    t = _fortran(tile, "tile")
    _raise(_lib.tc_round_host(t.shape[0], t.shape[1], t.ctypes.data, t.shape[0], level, int(lower)))


def quantize_block(b: np.ndarray, target: int) -> float:
    """tree.cpp:80-95; returns alpha"""
    t = _fortran(b, "b")
    al = C.c_double()
    _raise(_lib.tc_quantize_host(t.shape[0], t.shape[1], t.ctypes.data, t.shape[0], target, C.byref(al)))
    return al.value


def dequantize_block(b: np.ndarray, alpha: float, level: int):
    """tree.cpp:97-104"""
    t = _fortran(b, "b")
    _raise(_lib.tc_dequantize_host(t.shape[0], t.shape[1], t.ctypes.data, t.shape[0], level, float(alpha)))


def potrf_leaf(a: np.ndarray, level: int, acc: int = SINGLE):
    """kernels.cpp:42-69 in place; NotPositiveDefinite(local index)"""
    t = _fortran(a, "a")
    bad = C.c_int(-1)
    code = _lib.tc_potrf_leaf_host(t.shape[0], t.ctypes.data, t.shape[0], level, acc, C.byref(bad))
    if code == TC_NPD:
        raise NotPositiveDefinite(bad.value)
    _raise(code)


def trsm_leaf(b: np.ndarray, l: np.ndarray, level: int, acc: int = SINGLE):
    """kernels.cpp:71-92: B <- B L^-T in place; SingularDiagonal(local index)"""
    tb, tl = _fortran(b, "b"), _fortran(l, "l")
    bad = C.c_int(-1)
    code = _lib.tc_trsm_leaf_host(tb.shape[0], tb.shape[1], tb.ctypes.data, tb.shape[0], tl.ctypes.data,
                                  tl.shape[0], level, acc, C.byref(bad))
    if code == TC_SINGULAR:
        raise SingularDiagonal(bad.value)
    _raise(code)


def gemm_mixed(c: np.ndarray, a: np.ndarray, b: np.ndarray, alpha: float, beta: float, level: int,
               acc: int = SINGLE):
    """kernels.cpp:114-132: C <- beta C + alpha A B^T in place"""
    tc_, ta, tb = _fortran(c, "c"), _fortran(a, "a"), _fortran(b, "b")
    _raise(_lib.tc_gemm_mixed_host(tc_.shape[0], tc_.shape[1], ta.shape[1], tc_.ctypes.data, tc_.shape[0],
                                   ta.ctypes.data, ta.shape[0], tb.ctypes.data, tb.shape[0], float(alpha),
                                   float(beta), level, acc, 0))


def syrk_leaf(c: np.ndarray, a: np.ndarray, alpha: float, beta: float, level: int, acc: int = SINGLE):
    """kernels.cpp:94-112: lower(C) <- beta C + alpha A A^T in place"""
    tc_, ta = _fortran(c, "c"), _fortran(a, "a")
    _raise(_lib.tc_gemm_mixed_host(tc_.shape[0], tc_.shape[0], ta.shape[1], tc_.ctypes.data, tc_.shape[0],
                                   ta.ctypes.data, ta.shape[0], ta.ctypes.data, ta.shape[0], float(alpha),
                                   float(beta), level, acc, 1))


# ---------------------------------------------------------------- analysis.hpp
def spd_generate(n: int, seed: int) -> np.ndarray:
    """analysis.cpp:12-28, bit-identical (mt19937_64), Fortran float64."""
    a = np.empty((n, n), dtype=np.float64, order="F")
    _raise(_lib.tc_spd_generate_host(n, C.c_uint64(seed), a.ctypes.data, n))
    return a


def absmax_device(a_dev, m: int, n: int, stream=None) -> float:
    """max |A(i,j)| over the m x n column-major device block (NaN skipped)"""
    out = C.c_double()
    lda = a_dev.shape[1] if a_dev.dim() == 2 else m
    _raise(_lib.tc_absmax_device(m, n, _ptr(a_dev), lda, C.byref(out), _stream_ptr(stream)))
    return out.value


def spd_generate_device(n: int, seed: int, device="cuda"):
    """spd_generate(n, seed) straight into a device tensor (column-major
    memory, bit-identical to analysis.cpp:12-28)."""
    import torch
    t = torch.empty((n, n), dtype=torch.float64, device=device)
    _raise(_lib.tc_spd_generate_device(n, C.c_uint64(seed), _ptr(t), n, None))
    return t


def factorization_error_device(a_dev, l_dev, n: int | None = None, stream=None) -> float:
    """||A - L L^T||_F / ||A||_F in FP64 on the device (analysis.cpp:30-62)."""
    n = n or a_dev.shape[0]
    out = C.c_double()
    _raise(_lib.tc_factorization_error_device(n, _ptr(a_dev), _check_dev(a_dev, n, "a"), _ptr(l_dev),
                                              _check_dev(l_dev, n, "l"), C.byref(out), _stream_ptr(stream)))
    return out.value


def factorization_error(a: np.ndarray, l: np.ndarray) -> float:
    """host-array convenience wrapper over the device metric"""
    return factorization_error_device(to_device(a), to_device(l))


def potrs_device(l_dev, b_dev, n: int | None = None, stream=None):
    """A X = B with the factor L (lower, column-major); B (n x nrhs column-
    major, i.e. torch shape (nrhs, ldb)) is overwritten by X."""
    n = n or l_dev.shape[0]
    ldl = _check_dev(l_dev, n, "L")
    import torch
    if not (isinstance(b_dev, torch.Tensor) and b_dev.is_cuda and b_dev.dtype == torch.float64):
        raise InvalidArgument("B must be a CUDA float64 tensor")
    b2 = b_dev if b_dev.dim() == 2 else b_dev.view(1, -1)
    _raise(_lib.tc_potrs_device(n, _ptr(l_dev), ldl, _ptr(b2), b2.shape[1], b2.shape[0], _stream_ptr(stream)))
    return b_dev


def potrs_batch_device(l_list, b_list, n: int | None = None, stream=None):
    """the solves of independent systems in one launch sequence
    (tc_potrs_batch_device): l_list[k] factors (column-major device tensors
    of one shape), b_list[k] right-hand sides (nrhs, ldb) overwritten by X"""
    import torch
    k = len(l_list)
    if k != len(b_list):
        raise InvalidArgument("one right-hand side tensor per factor")
    if k == 0:
        return b_list
    n = n or l_list[0].shape[0]
    ldl = _check_dev(l_list[0], n, "L[0]")
    b2 = []
    for i, (l, b) in enumerate(zip(l_list, b_list)):
        if _check_dev(l, n, f"L[{i}]") != ldl or l.shape != l_list[0].shape:
            raise InvalidArgument(f"L[{i}] must have the shape of L[0]")
        if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == torch.float64 and b.is_contiguous()):
            raise InvalidArgument(f"B[{i}] must be a contiguous CUDA float64 tensor")
        b2.append(b if b.dim() == 2 else b.view(1, -1))
        if b2[-1].shape != b2[0].shape or b2[0].shape[1] < n:
            raise InvalidArgument(f"B[{i}] must be (nrhs, ldb >= n) like B[0]")
    pl = (C.c_void_p * k)(*[_ptr(x) for x in l_list])
    pb = (C.c_void_p * k)(*[_ptr(x) for x in b2])
    _raise(_lib.tc_potrs_batch_device(n, k, pl, ldl, pb, b2[0].shape[1], b2[0].shape[0], _stream_ptr(stream)))
    return b_list


def debug_gemm(gclass: str, m: int, n: int, k: int, lower: bool = False, beta: float = 1.0, exec_level: int = 0,
               iters: int = 20) -> float:
    """development: mean device microseconds of one grouped-GEMM launch"""
    out = C.c_float()
    _raise(_lib.tc_debug_gemm(GEMM_CLASSES.index(gclass), m, n, k, int(lower), float(beta), exec_level, iters,
                              C.byref(out)))
    return out.value


def set_global_option(key: str, value: int):
    """process-wide kernel settings (tc_set_global_option), for measurements"""
    _raise(_lib.tc_set_global_option(key.encode(), int(value)))


def gemm_problem_device(gclass: str, b16, b32, b64, ldw: int, m: int, n: int, k: int, a_r0: int, a_c0: int,
                        b_r0: int, b_c0: int, c_r0: int, c_c0: int, exec_level: int, lower: bool = False,
                        alpha: float = -1.0, beta: float = 1.0, stream=None):
    """one problem of a factorization GEMM class on caller level buffers
    (torch tensors or None, row-major with ld = ldw): the launch path the
    factorization graph uses (tc_gemm_problem_device)"""
    pr = (C.c_int * 11)(m, n, k, a_r0, a_c0, b_r0, b_c0, c_r0, c_c0, exec_level, int(bool(lower)))
    _raise(_lib.tc_gemm_problem_device(GEMM_CLASSES.index(gclass), None if b16 is None else _ptr(b16),
                                       None if b32 is None else _ptr(b32), None if b64 is None else _ptr(b64),
                                       int(ldw), pr, float(alpha), float(beta), _stream_ptr(stream)))


def debug_gemm_stamps():
    """ns offsets from kernel entry of CTA 0's phases in the last debug_gemm
    launch: setup, first TMA, first stage, accumulator, epilogue, exit"""
    arr = (C.c_uint64 * 15)()
    _raise(_lib.tc_debug_gemm_stamps(arr))
    return [int(arr[i]) - int(arr[0]) if arr[i] else None for i in range(1, 15)]


def solve_residual_device(a_dev, x_dev, b_dev, n: int | None = None, stream=None) -> float:
    n = n or a_dev.shape[0]
    out = C.c_double()
    _raise(_lib.tc_solve_residual_device(n, _ptr(a_dev), _check_dev(a_dev, n, "a"), _ptr(x_dev), _ptr(b_dev),
                                         C.byref(out), _stream_ptr(stream)))
    return out.value


@dataclass
class FactorReport:
    """analysis.hpp:15-27"""
    n: int = 0
    config: str = ""
    b: int = 0
    quantize: bool = True
    seed: int = 0
    status: str = ""
    detail: str = ""
    rel_error: float = float("nan")
    digits: float = float("nan")
    flops: FlopBreakdown = field(default_factory=FlopBreakdown)
    wall_ms: float = 0.0


def factor_matrix(a: np.ndarray, config, b: int, quantize: bool = True, plan: Plan | None = None) -> FactorReport:
    """analysis.cpp:122-155 on the device: copy A (the one permitted copy),
    factor it, map failures to a status, measure ||A - LL^T||/||A||."""
    import torch
    cfg = _cfg(config)
    n = a.shape[0]
    rep = FactorReport(n=n, config=cfg.to_string(), b=b, quantize=quantize)
    plan = plan or Plan(n, b, cfg, quantize)
    a_dev = to_device(a)
    l_dev = torch.empty_like(a_dev)
    l_dev.copy_(a_dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = plan.factor_device(a_dev, l_dev)
    rep.wall_ms = (time.perf_counter() - t0) * 1e3
    rep.flops = plan.run_flops()
    if st.status == "ok":
        rep.status = "ok"
        rep.rel_error = factorization_error_device(a_dev, l_dev)
        rep.digits = -math.log10(rep.rel_error) if rep.rel_error > 0 else float("inf")
    elif st.status == "singular-diagonal":
        raise SingularDiagonal(st.index, st.detail)
    else:
        rep.status, rep.detail = st.status, st.detail
    return rep


def _g17(v: float) -> str:
    """%.17g, NaN as "nan" (cli.cpp:19-24)"""
    if v != v:
        return "nan"
    return "%.17g" % v


CSV_HEADER = "n,config,leaf,quantize,seed,status,rel_error,digits,flops_f16,flops_f32,flops_f64,flops_total,wall_ms"


def write_csv(reports, out) -> None:
    """The reference's fixed CSV schema (cli.cpp:26-33, 123-127): header row,
    LF endings, doubles as %.17g, the config quoted.  `out` is a text stream."""
    out.write(CSV_HEADER + "\n")
    for r in reports:
        f = r.flops
        out.write("%d,\"%s\",%d,%d,%d,%s,%s,%s,%d,%d,%d,%d,%s\n" % (
            r.n, r.config, r.b, 1 if r.quantize else 0, r.seed, r.status, _g17(r.rel_error), _g17(r.digits),
            f.by_level[0], f.by_level[1], f.by_level[2], f.total(), _g17(r.wall_ms)))


def plan_report(n: int, b: int, config) -> str:
    """The `plan` subcommand's flop report (cli.cpp:52-86)."""
    cfg = _cfg(config)
    fb = flop_breakdown(n, b, cfg)
    t = float(fb.total())
    pct = (lambda f: 100.0 * f / t if t > 0 else 0.0)
    lines = ["n=%d leaf=%d config=%s total_flops=%d" % (n, b, cfg.to_string(), fb.total()), "", "per precision:"]
    for i, name in enumerate(("F16", "F32", "F64")):  # precision_name (precision.cpp:9-15)
        lines.append("  %-4s %20d  %6.2f%%" % (name, fb.by_level[i], pct(fb.by_level[i])))
    lines.append("per kernel:")
    for i, name in enumerate(("POTRF-leaf", "TRSM-leaf", "SYRK-leaf", "GEMM")):  # kernel_name (flops.cpp:5-12)
        lines.append("  %-10s %14d  %6.2f%%  (%d calls)" % (name, fb.by_kernel[i], pct(fb.by_kernel[i]), fb.calls[i]))
    lines.append("off-diagonal share (TRSM+SYRK+GEMM): %.2f%%" % pct(fb.by_kernel[1] + fb.by_kernel[2] + fb.by_kernel[3]))
    return "\n".join(lines) + "\n"


def accuracy_sweep(sizes, configs, b, seeds, quantize=True):
    """analysis.cpp:157-173: n-major, then config, then seed."""
    out = []
    for n in sizes:
        for cfg in configs:
            plan = Plan(n, b, _cfg(cfg), quantize)
            for s in seeds:
                r = factor_matrix(spd_generate(n, s), cfg, b, quantize, plan=plan)
                r.seed = s
                out.append(r)
    return out

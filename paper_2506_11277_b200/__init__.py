"""B200-native Ozaki-I FP64 GEMM (integer-slice emulation, arXiv 2506.11277).

Python mirror of the reference library's GEMM-path API (``ozmul``,
/root/reference/proj/include/ozmul/{scheme,analysis,slicing,mma_sim}.hpp)
over the C-ABI in ``include/ozgpu.h`` (``lib/libozgpu.so``).  Same names,
argument meanings and error classes as the reference:

    make_plan(cfg, k, slices_a, slices_b, schedule, strategy, mode, precision)
    multiply(a, b, cfg, plan) -> MultiplyResult(c, diagnostics)
    multiply_axpby(alpha, a, b, beta, c, cfg, plan)
    select_slices(kappa_a, kappa_b, width, u, s_max, options)
    scaling_profile(a, b)
    split_rows / split_cols / integer_gemm          (bit-exact debug hooks)
    chi / plan_levels / spare_carries / diagonal_flush_threshold /
    optimal_slice_width / max_inner_dim

All compute runs on the GPU through the native library; there is no CPU
fallback.  Importing the package fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

__all__ = [
    "ScheduleKind", "Accumulation", "SliceMode", "BlockOrientation", "MmaConfig",
    "MultiplyPlan", "Diagnostics", "MultiplyResult", "SliceSelection", "SelectOptions",
    "ScalingProfile", "SlicedMatrix", "OzmulError", "InvalidArgument", "DomainError",
    "DeviceError", "SelectionInfeasible", "MmaOverflowError", "make_plan", "multiply",
    "multiply_axpby", "multiply_device", "select_slices", "scaling_profile", "split_rows",
    "split_cols", "integer_gemm", "chi", "plan_levels", "spare_carries",
    "diagonal_flush_threshold", "optimal_slice_width", "max_inner_dim", "random_uniform",
    "gen_kappa_d", "kernel_launches", "library_path", "split_i8", "pair_planes", "gemm_fn",
    "multiply_device_multi", "min_exact_slices", "exact_gemm", "forward_error",
    "max_elementwise_error", "frobenius_norm", "normwise_gemm_error",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("OZGPU_LIB_OVERRIDE") or os.path.join(_HERE, "lib", "libozgpu.so")  # override: A/B tools


def library_path() -> str:
    return _LIB_PATH


if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the Ozaki-I path has no CPU fallback)")

_lib = ctypes.CDLL(_LIB_PATH)

# --------------------------------------------------------------------- ABI


class _Cfg(ctypes.Structure):
    _fields_ = [("input_width", ctypes.c_int), ("acc_width", ctypes.c_int)]


_MAX_LEVELS = 128


class _Plan(ctypes.Structure):
    _fields_ = [
        ("slices_a", ctypes.c_int), ("slices_b", ctypes.c_int), ("width", ctypes.c_int),
        ("schedule", ctypes.c_int), ("diag_sum_limit", ctypes.c_int),
        ("strategy", ctypes.c_int), ("mode", ctypes.c_int), ("precision", ctypes.c_int),
        ("acc_bits_used", ctypes.c_int), ("num_levels", ctypes.c_int),
        ("levels", ctypes.c_int * (2 * _MAX_LEVELS)), ("level_inexact_adds", ctypes.c_longlong),
        ("psi", ctypes.c_longlong),
    ]


class _Diag(ctypes.Structure):
    _fields_ = [
        ("products", ctypes.c_int64), ("integer_adds", ctypes.c_int64),
        ("float_adds", ctypes.c_int64), ("flushes", ctypes.c_int64),
        ("realized_psi", ctypes.c_longlong), ("planned_psi", ctypes.c_longlong),
        ("width", ctypes.c_int), ("acc_bits_used", ctypes.c_int),
    ]


class _Sel(ctypes.Structure):
    _fields_ = [("slices_a", ctypes.c_int), ("slices_b", ctypes.c_int), ("lhs", ctypes.c_double),
                ("target", ctypes.c_double), ("products", ctypes.c_int64),
                ("gap", ctypes.c_double)]


class _Prof(ctypes.Structure):
    _fields_ = [("kappa_a", ctypes.c_double), ("kappa_b", ctypes.c_double),
                ("a_has_zero_block", ctypes.c_int), ("b_has_zero_block", ctypes.c_int)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_DP = ctypes.POINTER(ctypes.c_double)


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_sig("ozgpu_last_error", ctypes.c_char_p)
_sig("ozgpu_version", ctypes.c_char_p)
_sig("ozgpu_create", ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P))
_sig("ozgpu_destroy", ctypes.c_int, _P)
_sig("ozgpu_kernel_launches", _I64, _P)
_sig("ozgpu_default_context", _P, ctypes.c_int)
_sig("ozgpu_optimal_slice_width", ctypes.c_int, _Cfg, _I64, ctypes.POINTER(ctypes.c_int))
_sig("ozgpu_max_inner_dim", ctypes.c_int, _Cfg, ctypes.POINTER(_I64))
_sig("ozgpu_chi", ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_I64))
_sig("ozgpu_spare_carries", ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
     ctypes.POINTER(_I64))
_sig("ozgpu_plan_levels", ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
     ctypes.POINTER(_Plan))
_sig("ozgpu_diagonal_flush_threshold", ctypes.c_int, _Cfg, ctypes.c_int, _I64,
     ctypes.POINTER(_I64))
_sig("ozgpu_make_plan", ctypes.c_int, _Cfg, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Plan))
_sig("ozgpu_select_slices", ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
     ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
     ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Sel))
_sig("ozgpu_scaling_profile", ctypes.c_int, _P, _I64, _I64, _I64, _DP, _I64, _DP, _I64,
     ctypes.POINTER(_Prof))
_sig("ozgpu_dgemm", ctypes.c_int, _P, _I64, _I64, _I64, _DP, _I64, _DP, _I64, _DP, _I64, _Cfg,
     ctypes.POINTER(_Plan), ctypes.POINTER(_Diag))
_sig("ozgpu_dgemm_axpby", ctypes.c_int, _P, _I64, _I64, _I64, ctypes.c_double, _DP, _I64, _DP,
     _I64, ctypes.c_double, _DP, _I64, _DP, _I64, _Cfg, ctypes.POINTER(_Plan),
     ctypes.POINTER(_Diag))
_sig("ozgpu_dgemm_device", ctypes.c_int, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _Cfg,
     ctypes.POINTER(_Plan), _P, _P, ctypes.POINTER(_Diag))
_sig("ozgpu_split", ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _DP, _I64, ctypes.c_int,
     ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int))
_sig("ozgpu_integer_gemm", ctypes.c_int, _P, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_int64),
     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
     ctypes.POINTER(ctypes.c_int64), _Cfg)

# ------------------------------------------------------------------ errors


class OzmulError(Exception):
    """Base class; ``code`` is the C-ABI error code."""
    code = 3


class InvalidArgument(OzmulError, ValueError):
    """std::invalid_argument in the reference."""
    code = 1


class DomainError(OzmulError, ArithmeticError):
    """std::domain_error in the reference (capacity / precision)."""
    code = 2


class DeviceError(OzmulError, RuntimeError):
    """CUDA failure or no sm_100 device (there is no CPU fallback)."""
    code = 3


class SelectionInfeasible(OzmulError, RuntimeError):
    """analysis.hpp:78-84: no (s_A, s_B) meets the target."""
    code = 4

    def __init__(self, msg, gap=0.0, best_lhs=0.0, target=0.0):
        super().__init__(msg)
        self.gap, self.best_lhs, self.target = gap, best_lhs, target


class MmaOverflowError(OzmulError, RuntimeError):
    """mma_sim.hpp:41-46: a simulated accumulator left I_T."""
    code = 5


class MatrixIOError(OzmulError, RuntimeError):
    """std::runtime_error of the reference's matrix file functions (io.cpp)."""
    code = 6


_ERRORS = {1: InvalidArgument, 2: DomainError, 3: DeviceError, 4: SelectionInfeasible,
           5: MmaOverflowError, 6: MatrixIOError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.ozgpu_last_error().decode()
        raise _ERRORS.get(rc, OzmulError)(msg)


# ------------------------------------------------------------------- types


class ScheduleKind(enum.IntEnum):
    FULL = 0      # kFull
    REDUCED = 1   # kReduced


class Accumulation(enum.IntEnum):
    FLOAT_PER_PRODUCT = 0  # kFloatPerProduct
    DIAGONAL_INTEGER = 1   # kDiagonalInteger
    LEVELLED_EXACT = 2     # kLevelledExact


class SliceMode(enum.IntEnum):
    TRUNCATE = 0  # kTruncate
    NEAREST = 1   # kNearest


class BlockOrientation(enum.IntEnum):
    ROWS = 0
    COLUMNS = 1


@dataclass(frozen=True)
class MmaConfig:
    """mma_sim.hpp:27-37."""
    input_width: int = 7
    acc_width: int = 31

    @staticmethod
    def int8_int32() -> "MmaConfig":
        return MmaConfig(7, 31)

    @staticmethod
    def int4_int32() -> "MmaConfig":
        return MmaConfig(3, 31)

    def _c(self) -> _Cfg:
        return _Cfg(self.input_width, self.acc_width)


@dataclass
class MultiplyPlan:
    """scheme.hpp:77-88 (Schedule and LevelPlan folded in)."""
    slices_a: int = 1
    slices_b: int = 1
    width: int = 7
    schedule: ScheduleKind = ScheduleKind.REDUCED
    diag_sum_limit: Optional[int] = None
    strategy: Accumulation = Accumulation.LEVELLED_EXACT
    mode: SliceMode = SliceMode.TRUNCATE
    precision: int = 53
    acc_bits_used: int = 0
    levels: List[Tuple[int, int]] = field(default_factory=list)
    level_inexact_adds: int = 0
    psi: int = 0

    @staticmethod
    def _from_c(p: _Plan) -> "MultiplyPlan":
        lv = [(p.levels[2 * i], p.levels[2 * i + 1]) for i in range(p.num_levels)]
        return MultiplyPlan(p.slices_a, p.slices_b, p.width, ScheduleKind(p.schedule),
                            p.diag_sum_limit if p.diag_sum_limit > 0 else None,
                            Accumulation(p.strategy), SliceMode(p.mode), p.precision,
                            p.acc_bits_used, lv, p.level_inexact_adds, p.psi)

    def _c(self) -> _Plan:
        p = _Plan()
        p.slices_a, p.slices_b, p.width = self.slices_a, self.slices_b, self.width
        p.schedule, p.strategy, p.mode = int(self.schedule), int(self.strategy), int(self.mode)
        p.diag_sum_limit = self.diag_sum_limit or 0
        p.precision, p.acc_bits_used = self.precision, self.acc_bits_used
        p.num_levels = len(self.levels)
        for i, (a, b) in enumerate(self.levels[:_MAX_LEVELS]):
            p.levels[2 * i], p.levels[2 * i + 1] = a, b
        p.level_inexact_adds, p.psi = self.level_inexact_adds, self.psi
        return p


@dataclass
class Diagnostics:
    """scheme.hpp:97-106."""
    products: int = 0
    integer_adds: int = 0
    float_adds: int = 0
    flushes: int = 0
    realized_psi: int = 0
    planned_psi: int = 0
    width: int = 0
    acc_bits_used: int = 0

    @staticmethod
    def _from_c(d: _Diag) -> "Diagnostics":
        return Diagnostics(d.products, d.integer_adds, d.float_adds, d.flushes, d.realized_psi,
                           d.planned_psi, d.width, d.acc_bits_used)


@dataclass
class MultiplyResult:
    c: np.ndarray
    diagnostics: Diagnostics


@dataclass
class SliceSelection:
    """analysis.hpp:86-92."""
    slices_a: int
    slices_b: int
    lhs: float
    target: float
    products: int


@dataclass
class SelectOptions:
    """analysis.hpp:94-100."""
    target: Optional[float] = None
    schedule: ScheduleKind = ScheduleKind.REDUCED
    strategy: Accumulation = Accumulation.LEVELLED_EXACT
    acc_bits_used: int = 31
    precision: int = 53


@dataclass
class ScalingProfile:
    """analysis.hpp:30-38 (scalar part)."""
    kappa_a: float
    kappa_b: float
    a_has_zero_block: bool
    b_has_zero_block: bool


@dataclass
class SlicedMatrix:
    """slicing.hpp:44-63: slices[l] is the l-th (most significant first) int64 slice."""
    orientation: BlockOrientation
    mode: SliceMode
    width: int
    scale_exponents: np.ndarray
    slices: np.ndarray  # [count, rows, cols] int64

    def slice_count(self) -> int:
        return int(self.slices.shape[0])

    def end_bit(self, index: int) -> int:
        last = (index + 1) * self.width
        return last - 1 if self.mode == SliceMode.NEAREST else last


# ----------------------------------------------------------------- context

_ctx_lock = threading.Lock()


def _ctx(device: Optional[int] = None) -> int:
    if device is None:
        device = int(os.environ.get("OZGPU_DEVICE", "0"))
    with _ctx_lock:
        c = _lib.ozgpu_default_context(device)
    if not c:
        raise DeviceError(_lib.ozgpu_last_error().decode())
    return c


def kernel_launches(device: Optional[int] = None) -> int:
    """Kernels this library launched through the default context so far."""
    return int(_lib.ozgpu_kernel_launches(_ctx(device)))


def version() -> str:
    return _lib.ozgpu_version().decode()


def _f64(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if a.ndim != 2:
        raise InvalidArgument("expected a 2-D matrix")
    return a


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_DP)


# ------------------------------------------------------------------ plan


def optimal_slice_width(cfg: MmaConfig, k: int) -> int:
    out = ctypes.c_int()
    _check(_lib.ozgpu_optimal_slice_width(cfg._c(), k, ctypes.byref(out)))
    return out.value


def max_inner_dim(cfg: MmaConfig) -> int:
    out = _I64()
    _check(_lib.ozgpu_max_inner_dim(cfg._c(), ctypes.byref(out)))
    return out.value


def chi(slices_a: int, slices_b: int) -> int:
    out = _I64()
    _check(_lib.ozgpu_chi(slices_a, slices_b, ctypes.byref(out)))
    return out.value


def spare_carries(first_diag: int, last_diag: int, width: int) -> int:
    out = _I64()
    _check(_lib.ozgpu_spare_carries(first_diag, last_diag, width, ctypes.byref(out)))
    return out.value


def plan_levels(precision: int, width: int, acc_bits_used: int, num_diagonals: int):
    """Returns (levels, inexact_adds) as scheme.cpp:64-95."""
    p = _Plan()
    _check(_lib.ozgpu_plan_levels(precision, width, acc_bits_used, num_diagonals, ctypes.byref(p)))
    return [(p.levels[2 * i], p.levels[2 * i + 1]) for i in range(p.num_levels)], \
        p.level_inexact_adds


def diagonal_flush_threshold(cfg: MmaConfig, width: int, k: int) -> int:
    out = _I64()
    _check(_lib.ozgpu_diagonal_flush_threshold(cfg._c(), width, k, ctypes.byref(out)))
    return out.value


def make_plan(cfg: MmaConfig, k: int, slices_a: int, slices_b: int,
              schedule: ScheduleKind = ScheduleKind.REDUCED,
              strategy: Accumulation = Accumulation.LEVELLED_EXACT,
              mode: SliceMode = SliceMode.TRUNCATE, precision: int = 53) -> MultiplyPlan:
    p = _Plan()
    _check(_lib.ozgpu_make_plan(cfg._c(), k, slices_a, slices_b, int(schedule), int(strategy),
                                int(mode), precision, ctypes.byref(p)))
    return MultiplyPlan._from_c(p)


# ------------------------------------------------------------- estimator


def select_slices(kappa_a: float, kappa_b: float, width: int, u: float, s_max: int,
                  options: Optional[SelectOptions] = None) -> SliceSelection:
    o = options or SelectOptions()
    s = _Sel()
    rc = _lib.ozgpu_select_slices(kappa_a, kappa_b, width, u, s_max, int(o.target is not None),
                                  o.target if o.target is not None else 0.0, int(o.schedule),
                                  int(o.strategy), o.acc_bits_used, o.precision, ctypes.byref(s))
    if rc == 4:
        raise SelectionInfeasible(_lib.ozgpu_last_error().decode(), s.gap, s.lhs, s.target)
    _check(rc)
    return SliceSelection(s.slices_a, s.slices_b, s.lhs, s.target, s.products)


def scaling_profile(a, b, device: Optional[int] = None) -> ScalingProfile:
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise InvalidArgument("scaling_profile: shape mismatch")
    out = _Prof()
    _check(_lib.ozgpu_scaling_profile(_ctx(device), a.shape[0], a.shape[1], b.shape[1], _dp(a),
                                      a.shape[1], _dp(b), b.shape[1], ctypes.byref(out)))
    return ScalingProfile(out.kappa_a, out.kappa_b, bool(out.a_has_zero_block),
                          bool(out.b_has_zero_block))


# ------------------------------------------------------------------ GEMM


_sig("ozgpu_dgemm_multi", ctypes.c_int, ctypes.POINTER(_P), ctypes.c_int, _I64, _I64, _I64, _DP,
     _I64, _DP, _I64, _DP, _I64, _Cfg, ctypes.POINTER(_Plan), ctypes.POINTER(_Diag))
_sig("ozgpu_device_contexts", ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
     ctypes.POINTER(_P))


def _slots(devices) -> Optional[list]:
    """Device slots for a sharded multiply: `devices` or $OZGPU_DEVICES."""
    if devices is None:
        env = os.environ.get("OZGPU_DEVICES", "")
        devices = [int(v) for v in env.split(",") if v.strip()] if env else None
    if devices is None or len(devices) < 2:
        return None
    arr = (ctypes.c_int * len(devices))(*devices)
    ctxs = (_P * len(devices))()
    _check(_lib.ozgpu_device_contexts(arr, len(devices), ctxs))
    return ctxs


def multiply(a, b, cfg: MmaConfig, plan: MultiplyPlan, device: Optional[int] = None,
             out: Optional[np.ndarray] = None, devices: Optional[List[int]] = None
             ) -> MultiplyResult:
    """scheme.cpp:219-361 on the GPU (host arrays in, host array out).

    `out` (optional) receives C in place, e.g. a pinned buffer.  `devices`
    (or $OZGPU_DEVICES, e.g. "0,1,2,3"): shard C in 2-D tiles over these GPUs
    (ozgpu_dgemm_multi; a device may repeat: extra contexts on it)."""
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise InvalidArgument("multiply: shape mismatch")
    m, k = a.shape
    n = b.shape[1]
    if out is not None:
        if out.shape != (m, n) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise InvalidArgument("multiply: out must be a contiguous float64 m x n array")
        c = out
    else:
        c = np.empty((m, n), dtype=np.float64)
    d = _Diag()
    pc = plan._c()
    slots = _slots(devices) if device is None else None
    if slots is not None:
        _check(_lib.ozgpu_dgemm_multi(slots, len(slots), m, n, k, _dp(a), k, _dp(b), n, _dp(c),
                                      n, cfg._c(), ctypes.byref(pc), ctypes.byref(d)))
    else:
        _check(_lib.ozgpu_dgemm(_ctx(device), m, n, k, _dp(a), k, _dp(b), n, _dp(c), n, cfg._c(),
                                ctypes.byref(pc), ctypes.byref(d)))
    return MultiplyResult(c, Diagnostics._from_c(d))


def multiply_axpby(alpha: float, a, b, beta: float, c, cfg: MmaConfig, plan: MultiplyPlan,
                   device: Optional[int] = None) -> MultiplyResult:
    """scheme.cpp:363-372."""
    a, b, c = _f64(a), _f64(b), _f64(c)
    if c.shape != (a.shape[0], b.shape[1]) or a.shape[1] != b.shape[0]:
        raise InvalidArgument("multiply_axpby: shape mismatch")
    m, k = a.shape
    n = b.shape[1]
    out = np.empty((m, n), dtype=np.float64)
    d = _Diag()
    pc = plan._c()
    _check(_lib.ozgpu_dgemm_axpby(_ctx(device), m, n, k, alpha, _dp(a), k, _dp(b), n, beta,
                                  _dp(c), n, _dp(out), n, cfg._c(), ctypes.byref(pc),
                                  ctypes.byref(d)))
    return MultiplyResult(out, Diagnostics._from_c(d))


def gemm_fn(cfg: MmaConfig, slices_a: int, slices_b: int,
            schedule: ScheduleKind = ScheduleKind.REDUCED,
            strategy: Accumulation = Accumulation.LEVELLED_EXACT,
            mode: SliceMode = SliceMode.TRUNCATE, precision: int = 53,
            device: Optional[int] = None):
    """The operator hook (`GemmFn`, oracle.hpp:117, consumed by block_lu_solve,
    oracle.cpp:371): a callable (x, y) -> x @ y that makes its plan per call
    for the operands' inner dimension, as the reference's callers do
    (main.cpp:578-582, acceptance_test.cpp:278-282)."""
    def fn(x, y):
        x = _f64(x)
        plan = make_plan(cfg, x.shape[1], slices_a, slices_b, schedule, strategy, mode, precision)
        return multiply(x, y, cfg, plan, device=device).c
    return fn


def multiply_device(m: int, n: int, k: int, a_ptr: int, lda: int, b_ptr: int, ldb: int,
                    c_ptr: int, ldc: int, cfg: MmaConfig, plan: MultiplyPlan,
                    stream: int = 0, status_ptr: int = 0,
                    device: Optional[int] = None) -> Diagnostics:
    """Device-resident multiply (ozgpu_dgemm_device): enqueues on `stream`, no sync."""
    d = _Diag()
    pc = plan._c()
    _check(_lib.ozgpu_dgemm_device(_ctx(device), m, n, k, a_ptr, lda, b_ptr, ldb, c_ptr, ldc,
                                   cfg._c(), ctypes.byref(pc), stream or None,
                                   status_ptr or None, ctypes.byref(d)))
    return Diagnostics._from_c(d)


_sig("ozgpu_dgemm_device_multi", ctypes.c_int, ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int,
     _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _Cfg, ctypes.POINTER(_Plan), _P, _P,
     ctypes.POINTER(_Diag))


def multiply_device_multi(m: int, n: int, k: int, a_ptr: int, lda: int, b_ptr: int, ldb: int,
                          c_ptr: int, ldc: int, cfg: MmaConfig, plan: MultiplyPlan,
                          devices: List[int], src_device: int = 0, stream: int = 0,
                          status_ptr: int = 0) -> Diagnostics:
    """Device-resident multiply sharded in 2-D C tiles over `devices`
    (ozgpu_dgemm_device_multi): A / B / C live on `src_device`, remote
    contexts pull their panels over NVLink and push their C block back.
    Ordered on `stream` (of src_device), no sync; `status_ptr`: 0 or
    len(devices) device ints on src_device, one per block."""
    if not devices:
        raise InvalidArgument("multiply_device_multi: no devices")
    arr = (ctypes.c_int * len(devices))(*devices)
    ctxs = (_P * len(devices))()
    _check(_lib.ozgpu_device_contexts(arr, len(devices), ctxs))
    d = _Diag()
    pc = plan._c()
    _check(_lib.ozgpu_dgemm_device_multi(ctxs, len(devices), src_device, m, n, k, a_ptr, lda,
                                         b_ptr, ldb, c_ptr, ldc, cfg._c(), ctypes.byref(pc),
                                         stream or None, status_ptr or None, ctypes.byref(d)))
    return Diagnostics._from_c(d)


# ------------------------------------------------------------ debug hooks


def _split(x, width: int, count: int, mode: SliceMode, orientation: int,
           device: Optional[int]) -> SlicedMatrix:
    x = _f64(x)
    rows, cols = x.shape
    slices = np.zeros((max(count, 0), rows, cols), dtype=np.int64)
    scales = np.zeros(rows if orientation == 0 else cols, dtype=np.int32)
    _check(_lib.ozgpu_split(_ctx(device), orientation, rows, cols, _dp(x), cols, width, count,
                            int(mode), slices.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                            scales.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))
    return SlicedMatrix(BlockOrientation(orientation), SliceMode(mode), width, scales, slices)


def split_rows(a, width: int, count: int, mode: SliceMode = SliceMode.TRUNCATE,
               device: Optional[int] = None) -> SlicedMatrix:
    """slicing.cpp:67-132, one scale per row, on the GPU."""
    return _split(a, width, count, mode, 0, device)


def split_cols(b, width: int, count: int, mode: SliceMode = SliceMode.TRUNCATE,
               device: Optional[int] = None) -> SlicedMatrix:
    """slicing.cpp:67-132, one scale per column, on the GPU."""
    return _split(b, width, count, mode, 1, device)


def integer_gemm(x, y, cfg: MmaConfig, c=None, device: Optional[int] = None) -> np.ndarray:
    """mma_sim.cpp:76-125 on the GPU (tcgen05 int8 path when provably exact)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.int64))
    if x.shape[1] != y.shape[0]:
        raise InvalidArgument("integer_gemm: shape mismatch")
    m, k = x.shape
    n = y.shape[1]
    cp = None
    if c is not None:
        cp = np.ascontiguousarray(np.asarray(c, dtype=np.int64))
        if cp.shape != (m, n):
            raise InvalidArgument("integer_gemm: accumulator shape mismatch")
    out = np.zeros((m, n), dtype=np.int64)
    P = ctypes.POINTER(ctypes.c_int64)
    _check(_lib.ozgpu_integer_gemm(_ctx(device), m, k, n, x.ctypes.data_as(P),
                                   y.ctypes.data_as(P),
                                   cp.ctypes.data_as(P) if cp is not None else None,
                                   out.ctypes.data_as(P), cfg._c()))
    return out


_sig("ozgpu_split_i8", ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _DP, _I64, ctypes.c_int,
     ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int8), _I64, ctypes.POINTER(ctypes.c_int))
_sig("ozgpu_pair_planes", ctypes.c_int, _P, _I64, _I64, _I64, _DP, _I64, _DP, _I64, _Cfg,
     ctypes.POINTER(_Plan), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
     ctypes.c_int, _I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_int32))


def split_i8(x, width: int, count: int, orientation: BlockOrientation,
             mode: SliceMode = SliceMode.TRUNCATE, device: Optional[int] = None):
    """The production int8 slicer (what multiply() runs on its operands) ->
    (slices [count, blocks, ld] int8, K-major with a zero-filled tail, scales).
    Bit-exact against split_rows / split_cols (slicing.cpp:67-132)."""
    x = _f64(x)
    rows, cols = x.shape
    blocks, length = (rows, cols) if int(orientation) == 0 else (cols, rows)
    ld = max(128, -(-length // 128) * 128)
    out = np.empty((count, blocks, ld), dtype=np.int8)
    scales = np.zeros(blocks, dtype=np.int32)
    _check(_lib.ozgpu_split_i8(_ctx(device), int(orientation), rows, cols, _dp(x), cols, width,
                               count, int(mode), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
                               ld, scales.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))
    return out, scales


def pair_planes(a, b, cfg: MmaConfig, plan: MultiplyPlan, window=None,
                device: Optional[int] = None):
    """The production pair GEMM's int32 chunk planes (before the combine) ->
    (planes [nchunks, rows, cols] int32 over `window` = (r0, r1, c0, c1),
    default all of C; chunks [(d, l0, npairs)]): chunk c is the exact sum of
    integer_gemm(A_l, B_h) over its pairs (l0 + p, d + 2 - l0 - p)."""
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise InvalidArgument("pair_planes: shape mismatch")
    m, k = a.shape
    n = b.shape[1]
    r0, r1, c0, c1 = window if window is not None else (0, m, 0, n)
    pc = plan._c()
    nc = ctypes.c_int()
    _check(_lib.ozgpu_pair_planes(_ctx(device), m, n, k, _dp(a), k, _dp(b), n, cfg._c(),
                                  ctypes.byref(pc), ctypes.byref(nc), None, 0, 0, 0, 0, 0, None))
    table = (ctypes.c_int * (3 * max(nc.value, 1)))()
    planes = np.zeros((nc.value, r1 - r0, c1 - c0), dtype=np.int32)
    _check(_lib.ozgpu_pair_planes(_ctx(device), m, n, k, _dp(a), k, _dp(b), n, cfg._c(),
                                  ctypes.byref(pc), ctypes.byref(nc), table, nc.value,
                                  r0, r1, c0, c1,
                                  planes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    chunks = [(table[3 * c], table[3 * c + 1], table[3 * c + 2]) for c in range(nc.value)]
    return planes, chunks


# -------------------------------------------------------------- generators


_gen = None


def _genlib():
    """lib/libozgen.so (include/ozgen.h): input generation, not the GEMM path."""
    global _gen
    if _gen is None:
        path = os.path.join(_HERE, "lib", "libozgen.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with __graft_entry__.build()")
        g = ctypes.CDLL(path)
        g.ozgen_random_uniform.restype = None
        g.ozgen_random_uniform.argtypes = [_I64, _I64, ctypes.c_uint64, ctypes.c_double,
                                           ctypes.c_double, _DP]
        g.ozgen_gen_kappa_d.restype = None
        g.ozgen_gen_kappa_d.argtypes = [_I64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int,
                                        _DP, _DP]
        _gen = g
    return _gen


def random_uniform(m: int, n: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """generators.cpp:176-182 (identical bytes to the reference generator)."""
    out = np.empty((m, n), dtype=np.float64)
    _genlib().ozgen_random_uniform(m, n, seed, lo, hi, _dp(out))
    return out


def gen_kappa_d(n: int, kappa_d: float, seed: int, rotate: bool):
    """generators.cpp:103-140."""
    a = np.empty((n, n), dtype=np.float64)
    b = np.empty((n, n), dtype=np.float64)
    _genlib().ozgen_gen_kappa_d(n, kappa_d, seed, int(rotate), _dp(a), _dp(b))
    return a, b


# ------------------------------------------------- ozm1 matrix files (io.hpp)


class MatrixFormat(enum.IntEnum):
    HEX = 0  # kHex: 16 hex digits of the binary64 bit pattern (bit-exact)
    DEC = 1  # kDec: shortest round-trip decimal


_sig("ozgpu_matrix_file_shape", ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_I64),
     ctypes.POINTER(_I64))
_sig("ozgpu_read_matrix_file", ctypes.c_int, ctypes.c_char_p, ctypes.c_int, _I64, _I64, _DP)
_sig("ozgpu_write_matrix_file", ctypes.c_int, ctypes.c_char_p, ctypes.c_int, _I64, _I64, _DP,
     _I64)


def read_matrix_file(path, fmt: MatrixFormat = MatrixFormat.HEX) -> np.ndarray:
    """read_matrix_file (io.hpp:33): an "ozm1 <rows> <cols>" file -> row-major f64."""
    rows, cols = _I64(), _I64()
    _check(_lib.ozgpu_matrix_file_shape(os.fsencode(path), ctypes.byref(rows), ctypes.byref(cols)))
    out = np.empty((rows.value, cols.value), dtype=np.float64)
    _check(_lib.ozgpu_read_matrix_file(os.fsencode(path), int(fmt), rows.value, cols.value,
                                       _dp(out)))
    return out


def write_matrix_file(path, a, fmt: MatrixFormat = MatrixFormat.HEX) -> None:
    """write_matrix_file (io.hpp:35)."""
    a = _f64(a)
    _check(_lib.ozgpu_write_matrix_file(os.fsencode(path), int(fmt), a.shape[0], a.shape[1],
                                        _dp(a), a.shape[1]))


# ------------------------------------------------------------ stage timing

_sig("ozgpu_set_stage_timing", ctypes.c_int, _P, ctypes.c_int)
_sig("ozgpu_stage_times", ctypes.c_int, _P, ctypes.POINTER(ctypes.c_double),
     ctypes.POINTER(_I64), ctypes.c_int)


def set_stage_timing(enable: bool, device: Optional[int] = None) -> None:
    """Record CUDA events around slicing / pair GEMMs / combine of each multiply."""
    _check(_lib.ozgpu_set_stage_timing(_ctx(device), int(enable)))


def stage_times(reset: bool = True, device: Optional[int] = None):
    """(slicing_ms, gemm_ms, combine_ms, calls) accumulated since the last reset."""
    ms = (ctypes.c_double * 3)()
    calls = _I64()
    _check(_lib.ozgpu_stage_times(_ctx(device), ms, ctypes.byref(calls), int(reset)))
    return ms[0], ms[1], ms[2], calls.value


# ------------------------------------------------ analysis helpers (GPU)

_sig("ozgpu_block_ratios", ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _DP, _I64, _DP,
     ctypes.POINTER(ctypes.c_int))
_sig("ozgpu_fp64_gemm", ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _I64, _DP, _I64, _DP, _I64,
     _DP, _I64)


def block_ratios(x, orientation: BlockOrientation, device: Optional[int] = None):
    """analysis.cpp:25-47 on the GPU -> (ratios, has_zero_block)."""
    x = _f64(x)
    nb = x.shape[0] if int(orientation) == 0 else x.shape[1]
    out = np.ones(nb, dtype=np.float64)
    z = ctypes.c_int()
    _check(_lib.ozgpu_block_ratios(_ctx(device), int(orientation), x.shape[0], x.shape[1], _dp(x),
                                   x.shape[1], _dp(out), ctypes.byref(z)))
    return out, bool(z.value)


def kappa(x, orientation: BlockOrientation, device: Optional[int] = None) -> float:
    """analysis.cpp:51-56: 2 * max(1, worst max/min-nonzero ratio)."""
    r, _ = block_ratios(x, orientation, device)
    return 2.0 * max(1.0, float(r.max()) if r.size else 1.0)


def abs_product(a, b, device: Optional[int] = None) -> np.ndarray:
    """|A||B| in binary64 with the reference's summation order (matrix.cpp:31-41)."""
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise InvalidArgument("abs_product: shape mismatch")
    out = np.empty((a.shape[0], b.shape[1]))
    _check(_lib.ozgpu_fp64_gemm(_ctx(device), 1, a.shape[0], a.shape[1], b.shape[1], _dp(a),
                                a.shape[1], _dp(b), b.shape[1], _dp(out), b.shape[1]))
    return out


_sig("ozgpu_min_exact_slices", ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _DP, _I64, ctypes.c_int,
     ctypes.c_int, ctypes.POINTER(ctypes.c_int))
_sig("ozgpu_exact_gemm", ctypes.c_int, _P, _I64, _I64, _I64, _DP, _I64, _DP, _I64, _DP, _I64)
_sig("ozgpu_error_metrics", ctypes.c_int, _P, _I64, _I64, _DP, _I64, _DP, _I64,
     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double))


def min_exact_slices(x, width: int, orientation: BlockOrientation,
                     mode: SliceMode = SliceMode.TRUNCATE, device: Optional[int] = None) -> int:
    """slicing.cpp:212-249 on the GPU."""
    x = _f64(x)
    out = ctypes.c_int()
    _check(_lib.ozgpu_min_exact_slices(_ctx(device), int(orientation), x.shape[0], x.shape[1],
                                       _dp(x), x.shape[1], width, int(mode), ctypes.byref(out)))
    return out.value


def exact_gemm(a, b, device: Optional[int] = None) -> np.ndarray:
    """exact_gemm(a, b).to_matrix() (oracle.cpp:223-232) on the GPU: RN(AB)
    entrywise, via error-free slices and the full pair schedule."""
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise InvalidArgument("exact_gemm: shape mismatch")
    out = np.empty((a.shape[0], b.shape[1]))
    _check(_lib.ozgpu_exact_gemm(_ctx(device), a.shape[0], b.shape[1], a.shape[1], _dp(a),
                                 a.shape[1], _dp(b), b.shape[1], _dp(out), b.shape[1]))
    return out


def _metrics(c, r, device):
    c = _f64(c)
    mx, ss = ctypes.c_double(), ctypes.c_double()
    if r is not None:
        r = _f64(r)
        if r.shape != c.shape:
            raise InvalidArgument("max_elementwise_error: shape mismatch")
    _check(_lib.ozgpu_error_metrics(_ctx(device), c.shape[0], c.shape[1], _dp(c), c.shape[1],
                                    _dp(r) if r is not None else None,
                                    r.shape[1] if r is not None else 0, ctypes.byref(mx),
                                    ctypes.byref(ss)))
    return mx.value, ss.value


def forward_error(computed: float, exact: float) -> float:
    """oracle.cpp:253-261 with the exact value given as a double (RN(exact))."""
    if exact == 0.0:
        return 0.0 if computed == 0.0 else float("inf")
    return abs(computed - exact) / abs(exact)


def max_elementwise_error(computed, exact, device: Optional[int] = None) -> float:
    """oracle.cpp:263-271 on the GPU, `exact` = RN(exact product) (e.g. from
    exact_gemm): max over entries of |c - e| / |e|.  Against the reference's
    unrounded ExactValue the per-entry error differs by at most ~1.1 u."""
    return _metrics(computed, exact, device)[0]


def frobenius_norm(x, device: Optional[int] = None) -> float:
    """oracle.cpp:64-68 on the GPU (deterministic tree order)."""
    import math
    return math.sqrt(_metrics(x, None, device)[1])


def normwise_gemm_error(dhat, dref, a, b, c, alpha: float, beta: float,
                        device: Optional[int] = None) -> float:
    """oracle.cpp:273-292 on the GPU; `dref` = RN(exact) as the reference's
    dexact.to_matrix()."""
    import math
    dhat = _f64(dhat)
    num = math.sqrt(_metrics(dhat, dref, device)[1])
    k = float(_f64(a).shape[1])
    denom = (abs(alpha) * math.sqrt(k + 2.0) * frobenius_norm(a, device) *
             frobenius_norm(b, device) + 2.0 * abs(beta) * frobenius_norm(c, device))
    if denom == 0.0:
        raise DomainError("normwise_gemm_error: zero denominator")
    return num / denom


def zeta(kappa_a: float, kappa_b: float, slices_a: int, slices_b: int, width: int) -> float:
    """analysis.cpp:70-77."""
    import math
    if not (kappa_a > 0 and kappa_b > 0):
        raise InvalidArgument("zeta: kappas must be positive")
    return (math.ldexp(kappa_a, -slices_a * width) + math.ldexp(kappa_b, -slices_b * width) +
            math.ldexp(kappa_a * kappa_b, -(slices_a + slices_b) * width))


def gamma_factor(n: int, u: float) -> float:
    """analysis.cpp:79-84."""
    if n < 0:
        raise InvalidArgument("gamma_factor: n must be >= 0")
    nu = float(n) * u
    if nu >= 1.0:
        raise DomainError("gamma_factor: n*u >= 1, bound is meaningless")
    return nu / (1.0 - nu)


@dataclass
class ErrorReport:
    """analysis.hpp:52-64."""
    kappa_a: float
    kappa_b: float
    zeta_ab: float
    gamma_psi: float
    coefficient: float
    first_order_coefficient: float
    kind: str
    bound: np.ndarray


def error_bound(a, b, plan: MultiplyPlan, u: float = 2.0 ** -53,
                device: Optional[int] = None) -> ErrorReport:
    """analysis.cpp:86-131: coefficient * |A||B| * (1 + 8u), |A||B| on the GPU."""
    import math
    prof = scaling_profile(a, b, device)
    t, sa, sb = plan.width, plan.slices_a, plan.slices_b
    z = zeta(prof.kappa_a, prof.kappa_b, sa, sb, t)
    g = gamma_factor(plan.psi, u)
    if plan.schedule == ScheduleKind.FULL:
        kind, coef = "full", z + g * (1.0 + z)
    else:
        if sa <= sb:
            kind, cut = "reduced_a_le_b", math.ldexp(float(sa) * prof.kappa_a * prof.kappa_b, -sb * t)
        else:
            kind, cut = "reduced_a_gt_b", math.ldexp(float(sb) * prof.kappa_a * prof.kappa_b, -sa * t)
        gn = gamma_factor(plan.psi + 1, u)
        coef = z + cut + gn * (1.0 + z + cut)
    first = (math.ldexp(prof.kappa_a, -sa * t) + math.ldexp(prof.kappa_b, -sb * t) +
             float(plan.psi) * u)
    bound = abs_product(a, b, device) * (coef * (1.0 + 8.0 * u))
    return ErrorReport(prof.kappa_a, prof.kappa_b, z, g, coef, first, kind, bound)

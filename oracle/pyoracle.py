"""ctypes loaders for the two CPU oracles (TEST INFRASTRUCTURE ONLY).

* ``port()``  -- oracle/lib/liboz_oracle.so, the plain-C restatement (ozoracle.c)
* ``ref()``   -- oracle/_ref/libozref.so, the UNMODIFIED reference compiled from
                 its own sources (oracle/Makefile) behind a C-ABI (ref_capi.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module, and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "lib", "liboz_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libozref.so")

_DP = ctypes.POINTER(ctypes.c_double)
_LP = ctypes.POINTER(ctypes.c_int64)
_IP = ctypes.POINTER(ctypes.c_int)
_I64 = ctypes.c_int64
_port = None
_ref = None


def build() -> None:
    """make -C oracle (reference targets only when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _dp(a):
    return a.ctypes.data_as(_DP)


def _lp(a):
    return a.ctypes.data_as(_LP)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            build()
        lib = ctypes.CDLL(PORT_PATH)
        lib.ozo_optimal_slice_width.restype = ctypes.c_int
        lib.ozo_optimal_slice_width.argtypes = [ctypes.c_int, ctypes.c_int, _I64]
        lib.ozo_chi.restype = _I64
        lib.ozo_chi.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.ozo_spare_carries.restype = _I64
        lib.ozo_spare_carries.argtypes = [ctypes.c_int] * 3
        lib.ozo_plan_levels.restype = ctypes.c_int
        lib.ozo_plan_levels.argtypes = [ctypes.c_int] * 4 + [_IP, ctypes.c_int]
        lib.ozo_max_diag_sum.restype = ctypes.c_int
        lib.ozo_max_diag_sum.argtypes = [ctypes.c_int] * 4
        lib.ozo_split.restype = ctypes.c_int
        lib.ozo_split.argtypes = [ctypes.c_int, _I64, _I64, _DP, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, _LP, _IP]
        lib.ozo_integer_gemm.restype = ctypes.c_int
        lib.ozo_integer_gemm.argtypes = [_I64, _I64, _I64, _LP, _LP, _LP, ctypes.c_int,
                                         ctypes.c_int]
        lib.ozo_round_words.restype = ctypes.c_double
        lib.ozo_round_words.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                                        ctypes.c_long]
        lib.ozo_multiply_exact.restype = ctypes.c_int
        lib.ozo_multiply_exact.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP] + [ctypes.c_int] * 6
        lib.ozo_scaling_profile.restype = None
        lib.ozo_scaling_profile.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP, _DP, _IP, _IP]
        lib.ozo_select_slices.restype = ctypes.c_int
        lib.ozo_select_slices.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, _IP, _IP, _DP, _DP, _LP,
                                          _DP]
        lib.ozo_random_uniform.restype = None
        lib.ozo_random_uniform.argtypes = [_I64, _I64, ctypes.c_uint64, ctypes.c_double,
                                           ctypes.c_double, _DP]
        lib.ozo_gen_kappa_d.restype = None
        lib.ozo_gen_kappa_d.argtypes = [_I64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int,
                                        _DP, _DP]
        _port = lib
    return _port


def have_ref() -> bool:
    if not os.path.exists(REF_PATH) and os.path.isdir("/root/reference/proj"):
        build()
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise RuntimeError("oracle/_ref/libozref.so is not built and /root/reference is absent")
        lib = ctypes.CDLL(REF_PATH)
        lib.ozref_last_error.restype = ctypes.c_char_p
        lib.ozref_multiply.restype = ctypes.c_int
        lib.ozref_multiply.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP] + [ctypes.c_int] * 9 + [_LP]
        lib.ozref_multiply_width.restype = ctypes.c_int
        lib.ozref_multiply_width.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP] + [ctypes.c_int] * 3
        lib.ozref_multiply_blocks.restype = ctypes.c_int
        lib.ozref_multiply_blocks.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP] + \
            [ctypes.c_int] * 7 + [_LP, ctypes.c_int, _DP]
        lib.ozref_split.restype = ctypes.c_int
        lib.ozref_split.argtypes = [ctypes.c_int, _I64, _I64, _DP, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _LP, _IP]
        lib.ozref_reconstruct.restype = ctypes.c_int
        lib.ozref_reconstruct.argtypes = [ctypes.c_int, _I64, _I64, _DP, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, _DP]
        lib.ozref_min_exact_slices.restype = ctypes.c_int
        lib.ozref_min_exact_slices.argtypes = [ctypes.c_int, _I64, _I64, _DP, ctypes.c_int,
                                               ctypes.c_int, _IP]
        lib.ozref_integer_gemm.restype = ctypes.c_int
        lib.ozref_integer_gemm.argtypes = [_I64, _I64, _I64, _LP, _LP, _LP, ctypes.c_int,
                                           ctypes.c_int]
        lib.ozref_make_plan.restype = ctypes.c_int
        lib.ozref_make_plan.argtypes = [_I64] + [ctypes.c_int] * 8 + [
            _IP, _IP, ctypes.POINTER(ctypes.c_longlong), _IP, _IP, ctypes.c_int]
        lib.ozref_plan_levels.restype = ctypes.c_int
        lib.ozref_plan_levels.argtypes = [ctypes.c_int] * 4 + [_IP, _IP, ctypes.c_int]
        lib.ozref_chi.restype = ctypes.c_longlong
        lib.ozref_chi.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.ozref_select_slices.restype = ctypes.c_int
        lib.ozref_select_slices.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                            ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, _IP, _IP, _DP, _DP,
                                            ctypes.POINTER(ctypes.c_longlong), _DP]
        lib.ozref_scaling_profile.restype = ctypes.c_int
        lib.ozref_scaling_profile.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP, _DP, _IP, _IP]
        lib.ozref_error_bound.restype = ctypes.c_int
        lib.ozref_error_bound.argtypes = [_I64, _I64, _I64, _DP, _DP] + [ctypes.c_int] * 6 + \
            [_DP, _DP]
        lib.ozref_exact_gemm.restype = ctypes.c_int
        lib.ozref_exact_gemm.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP]
        lib.ozref_fp64_gemm.restype = ctypes.c_int
        lib.ozref_fp64_gemm.argtypes = [ctypes.c_int, _I64, _I64, _I64, _DP, _DP, _DP]
        lib.ozref_error_metrics.restype = ctypes.c_int
        lib.ozref_error_metrics.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP, _DP, _DP]
        lib.ozref_exact_gemm_axpby.restype = ctypes.c_int
        lib.ozref_exact_gemm_axpby.argtypes = [_I64, _I64, _I64, ctypes.c_double, _DP, _DP,
                                               ctypes.c_double, _DP, _DP]
        lib.ozref_multiply_axpby.restype = ctypes.c_int
        lib.ozref_multiply_axpby.argtypes = [_I64, _I64, _I64, ctypes.c_double, _DP, _DP,
                                             ctypes.c_double, _DP, _DP] + [ctypes.c_int] * 6
        lib.ozref_random_uniform.restype = None
        lib.ozref_random_uniform.argtypes = [_I64, _I64, ctypes.c_uint64, ctypes.c_double,
                                             ctypes.c_double, _DP]
        lib.ozref_gen_kappa_d.restype = ctypes.c_int
        lib.ozref_gen_kappa_d.argtypes = [_I64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int,
                                          _DP, _DP]
        _ref = lib
    return _ref


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _rc(code: int):
    if code:
        raise RefError(code, ref().ozref_last_error().decode())


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


# ---------------------------------------------------------- reference (GMP)


def ref_multiply(a, b, sa: int, sb: int, schedule: int = 1, strategy: int = 2, mode: int = 0,
                 precision: int = 53, diag_sum_limit: int = 0, cfg=(7, 31)):
    """Reference multiply() (scheme.cpp:219-361) -> (C, diag[8])."""
    a, b = _f64(a), _f64(b)
    m, k = a.shape
    n = b.shape[1]
    c = np.zeros((m, n))
    diag = np.zeros(8, dtype=np.int64)
    _rc(ref().ozref_multiply(m, n, k, _dp(a), _dp(b), _dp(c), sa, sb, schedule, strategy, mode,
                             precision, diag_sum_limit, cfg[0], cfg[1], _lp(diag)))
    return c, diag


def ref_multiply_blocks(a, b, sa: int, sb: int, blocks: Sequence[Tuple[int, int, int, int]],
                        threads: int, schedule: int = 1, strategy: int = 2, mode: int = 0,
                        precision: int = 53):
    """Reference multiply() on C blocks, one std::thread per block -> (C, seconds)."""
    a, b = _f64(a), _f64(b)
    m, k = a.shape
    n = b.shape[1]
    c = np.full((m, n), np.nan)
    blk = np.ascontiguousarray(np.asarray(blocks, dtype=np.int64).reshape(-1, 4))
    secs = ctypes.c_double()
    _rc(ref().ozref_multiply_blocks(m, n, k, _dp(a), _dp(b), _dp(c), sa, sb, schedule, strategy,
                                    mode, precision, len(blk), _lp(blk), threads,
                                    ctypes.byref(secs)))
    return c, secs.value


def ref_split(x, orientation: int, width: int, count: int, mode: int = 0):
    x = _f64(x)
    rows, cols = x.shape
    sl = np.zeros((count, rows, cols), dtype=np.int64)
    sc = np.zeros(rows if orientation == 0 else cols, dtype=np.int32)
    _rc(ref().ozref_split(orientation, rows, cols, _dp(x), width, count, mode, _lp(sl),
                          sc.ctypes.data_as(_IP)))
    return sc, sl


def ref_min_exact_slices(x, orientation: int, width: int, mode: int = 0) -> int:
    x = _f64(x)
    out = ctypes.c_int()
    _rc(ref().ozref_min_exact_slices(orientation, x.shape[0], x.shape[1], _dp(x), width, mode,
                                     ctypes.byref(out)))
    return out.value


def ref_integer_gemm(x, y, t_in: int = 7, t_acc: int = 31):
    x = np.ascontiguousarray(x, dtype=np.int64)
    y = np.ascontiguousarray(y, dtype=np.int64)
    out = np.zeros((x.shape[0], y.shape[1]), dtype=np.int64)
    _rc(ref().ozref_integer_gemm(x.shape[0], x.shape[1], y.shape[1], _lp(x), _lp(y), _lp(out),
                                 t_in, t_acc))
    return out


def ref_make_plan(k, sa, sb, schedule=1, strategy=2, mode=0, precision=53, cfg=(7, 31)):
    w, acc, nl = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    psi = ctypes.c_longlong()
    lv = (ctypes.c_int * 512)()
    _rc(ref().ozref_make_plan(k, sa, sb, schedule, strategy, mode, precision, cfg[0], cfg[1],
                              ctypes.byref(w), ctypes.byref(acc), ctypes.byref(psi),
                              ctypes.byref(nl), lv, 256))
    levels = [(lv[2 * i], lv[2 * i + 1]) for i in range(nl.value)]
    return {"width": w.value, "acc_bits_used": acc.value, "psi": psi.value, "levels": levels}


def ref_plan_levels(precision, width, acc_bits_used, diagonals):
    nl = ctypes.c_int()
    lv = (ctypes.c_int * 1024)()
    _rc(ref().ozref_plan_levels(precision, width, acc_bits_used, diagonals, ctypes.byref(nl), lv,
                                512))
    return [(lv[2 * i], lv[2 * i + 1]) for i in range(nl.value)]


def ref_select_slices(kappa_a, kappa_b, width, u, s_max, target=None, schedule=1, strategy=2,
                      acc_bits_used=31, precision=53):
    sa, sb = ctypes.c_int(), ctypes.c_int()
    lhs, tgt, gap = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    prod = ctypes.c_longlong()
    code = ref().ozref_select_slices(kappa_a, kappa_b, width, u, s_max, int(target is not None),
                                     target or 0.0, schedule, strategy, acc_bits_used, precision,
                                     ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(lhs),
                                     ctypes.byref(tgt), ctypes.byref(prod), ctypes.byref(gap))
    if code == 4:
        return {"infeasible": True, "gap": gap.value, "lhs": lhs.value, "target": tgt.value}
    _rc(code)
    return {"slices_a": sa.value, "slices_b": sb.value, "lhs": lhs.value, "target": tgt.value,
            "products": prod.value}


def ref_scaling_profile(a, b):
    a, b = _f64(a), _f64(b)
    ka, kb = ctypes.c_double(), ctypes.c_double()
    za, zb = ctypes.c_int(), ctypes.c_int()
    _rc(ref().ozref_scaling_profile(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b),
                                    ctypes.byref(ka), ctypes.byref(kb), ctypes.byref(za),
                                    ctypes.byref(zb)))
    return ka.value, kb.value, bool(za.value), bool(zb.value)


def ref_error_bound(a, b, sa, sb, schedule=1, strategy=2, mode=0, precision=53, want_bound=True):
    a, b = _f64(a), _f64(b)
    coef = ctypes.c_double()
    bound = np.zeros((a.shape[0], b.shape[1])) if want_bound else None
    _rc(ref().ozref_error_bound(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b), sa, sb,
                                schedule, strategy, mode, precision, ctypes.byref(coef),
                                _dp(bound) if want_bound else None))
    return coef.value, bound


def ref_exact_gemm(a, b):
    a, b = _f64(a), _f64(b)
    out = np.zeros((a.shape[0], b.shape[1]))
    _rc(ref().ozref_exact_gemm(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b), _dp(out)))
    return out


def ref_fp64_gemm(a, b, absolute=True):
    """Reference abs_product (absolute) / gemm_reference (matrix.cpp:31-54)."""
    a, b = _f64(a), _f64(b)
    out = np.zeros((a.shape[0], b.shape[1]))
    _rc(ref().ozref_fp64_gemm(int(absolute), a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b),
                              _dp(out)))
    return out


def ref_error_metrics(a, b, computed):
    """Reference max_elementwise_error and normwise_gemm_error (alpha 1, beta
    0) of `computed` against exact_gemm(a, b) (oracle.cpp:263-292)."""
    a, b, computed = _f64(a), _f64(b), _f64(computed)
    mx, nw = ctypes.c_double(), ctypes.c_double()
    _rc(ref().ozref_error_metrics(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b),
                                  _dp(computed), ctypes.byref(mx), ctypes.byref(nw)))
    return mx.value, nw.value


def ref_multiply_axpby(alpha, a, b, beta, c, sa, sb, schedule=1, strategy=2, mode=0,
                       precision=53):
    a, b, c = _f64(a), _f64(b), _f64(c)
    out = np.zeros_like(c)
    _rc(ref().ozref_multiply_axpby(a.shape[0], b.shape[1], a.shape[1], alpha, _dp(a), _dp(b),
                                   beta, _dp(c), _dp(out), sa, sb, schedule, strategy, mode,
                                   precision))
    return out


def ref_random_uniform(m, n, seed, lo=0.0, hi=1.0):
    out = np.empty((m, n))
    ref().ozref_random_uniform(m, n, seed, lo, hi, _dp(out))
    return out


def _ozm_tool():
    tool = os.path.join(os.path.dirname(REF_PATH), "ozm_tool")
    if not os.path.exists(tool):
        have_ref()
    if not os.path.exists(tool):
        raise RuntimeError("oracle/_ref/ozm_tool is not built")
    return tool


def ref_write_matrix_file(path, a, fmt=0):
    """The reference's write_matrix_file (io.cpp:97-103) via oracle/_ref/ozm_tool
    (a separate process: the reference's stream code is not called in-process);
    fmt 0 hex, 1 decimal."""
    import subprocess
    import tempfile
    a = _f64(a)
    with tempfile.NamedTemporaryFile(suffix=".f64") as raw:
        raw.write(a.tobytes())
        raw.flush()
        subprocess.run([_ozm_tool(), "w", "hex" if fmt == 0 else "dec", str(a.shape[0]),
                        str(a.shape[1]), raw.name, str(path)], check=True)


def ref_read_matrix_file(path, fmt=0):
    """The reference's read_matrix_file (io.cpp:65-69) -> ndarray."""
    import subprocess
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".f64") as raw:
        r = subprocess.run([_ozm_tool(), "r", "hex" if fmt == 0 else "dec", str(path), raw.name],
                           check=True, capture_output=True, text=True)
        rows, cols = (int(v) for v in r.stdout.split())
        return np.fromfile(raw.name, dtype=np.float64).reshape(rows, cols)


def ref_gen_kappa_d(n, kappa_d, seed, rotate):
    a, b = np.empty((n, n)), np.empty((n, n))
    _rc(ref().ozref_gen_kappa_d(n, kappa_d, seed, int(rotate), _dp(a), _dp(b)))
    return a, b


# -------------------------------------------------------------- C port


def port_split(x, orientation: int, width: int, count: int, mode: int = 0):
    x = _f64(x)
    rows, cols = x.shape
    sl = np.zeros((count, rows, cols), dtype=np.int64)
    sc = np.zeros(rows if orientation == 0 else cols, dtype=np.int32)
    rc = port().ozo_split(orientation, rows, cols, _dp(x), width, count, mode, _lp(sl),
                          sc.ctypes.data_as(_IP))
    if rc:
        raise RefError(rc, "ozo_split")
    return sc, sl


def port_integer_gemm(x, y, t_in: int = 7, t_acc: int = 31):
    x = np.ascontiguousarray(x, dtype=np.int64)
    y = np.ascontiguousarray(y, dtype=np.int64)
    out = np.zeros((x.shape[0], y.shape[1]), dtype=np.int64)
    rc = port().ozo_integer_gemm(x.shape[0], x.shape[1], y.shape[1], _lp(x), _lp(y), _lp(out),
                                 t_in, t_acc)
    if rc:
        raise RefError(rc, "ozo_integer_gemm")
    return out


def port_multiply_exact(a, b, sa, sb, schedule=1, diag_sum_limit=0, mode=0, width=None):
    a, b = _f64(a), _f64(b)
    m, k = a.shape
    n = b.shape[1]
    if width is None:
        width = port().ozo_optimal_slice_width(7, 31, max(k, 1))
    c = np.zeros((m, n))
    rc = port().ozo_multiply_exact(m, n, k, _dp(a), _dp(b), _dp(c), sa, sb, schedule,
                                   diag_sum_limit, mode, width)
    if rc:
        raise RefError(rc, "ozo_multiply_exact")
    return c


def port_plan_levels(precision, width, acc_bits_used, diagonals):
    lv = (ctypes.c_int * 1024)()
    nl = port().ozo_plan_levels(precision, width, acc_bits_used, diagonals, lv, 512)
    return [(lv[2 * i], lv[2 * i + 1]) for i in range(nl)]


def port_select_slices(kappa_a, kappa_b, width, u, s_max, target=None, schedule=1, strategy=2,
                       acc_bits_used=31, precision=53):
    sa, sb = ctypes.c_int(), ctypes.c_int()
    lhs, tgt, gap = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    prod = ctypes.c_int64()
    code = port().ozo_select_slices(kappa_a, kappa_b, width, u, s_max, int(target is not None),
                                    target or 0.0, schedule, strategy, acc_bits_used, precision,
                                    ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(lhs),
                                    ctypes.byref(tgt), ctypes.byref(prod), ctypes.byref(gap))
    if code == 4:
        return {"infeasible": True, "gap": gap.value, "lhs": lhs.value, "target": tgt.value}
    if code:
        raise RefError(code, "ozo_select_slices")
    return {"slices_a": sa.value, "slices_b": sb.value, "lhs": lhs.value, "target": tgt.value,
            "products": prod.value}


def port_scaling_profile(a, b):
    a, b = _f64(a), _f64(b)
    ka, kb = ctypes.c_double(), ctypes.c_double()
    za, zb = ctypes.c_int(), ctypes.c_int()
    port().ozo_scaling_profile(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b),
                               ctypes.byref(ka), ctypes.byref(kb), ctypes.byref(za),
                               ctypes.byref(zb))
    return ka.value, kb.value, bool(za.value), bool(zb.value)


def port_random_uniform(m, n, seed, lo=0.0, hi=1.0):
    out = np.empty((m, n))
    port().ozo_random_uniform(m, n, seed, lo, hi, _dp(out))
    return out


def port_gen_kappa_d(n, kappa_d, seed, rotate):
    a, b = np.empty((n, n)), np.empty((n, n))
    port().ozo_gen_kappa_d(n, kappa_d, seed, int(rotate), _dp(a), _dp(b))
    return a, b

"""The kernels' bit-level numerics (csrc/ozgpu_numeric.h), compiled for the
host, against the C restatement and Python big integers."""
import ctypes
import math
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def nt(tmp_path_factory):
    out = tmp_path_factory.mktemp("nt") / "libnt.so"
    subprocess.run(["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-I",
                    os.path.join(ROOT, "paper_2506_11277_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "numeric_shim.cpp"), "-o", str(out)],
                   check=True)
    lib = ctypes.CDLL(str(out))
    lib.nt_ldexp_rn.restype = ctypes.c_double
    lib.nt_ldexp_rn.argtypes = [ctypes.c_double, ctypes.c_long]
    lib.nt_accumulate_round.restype = ctypes.c_double
    lib.nt_accumulate_round.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_long]
    lib.nt_accumulate_words.restype = None
    lib.nt_accumulate_words.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]
    lib.nt_slices.restype = None
    lib.nt_slices.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, ctypes.c_void_p]
    return lib


def test_ldexp_rn_matches_libm(nt):
    rng = np.random.default_rng(1)
    for _ in range(20000):
        d = float(rng.integers(1, 2**56)) * (1 if rng.random() < 0.5 else -1)
        e = int(rng.integers(-1200, 1000))
        want = math.ldexp(d, e) if e < 1000 - 56 else math.copysign(math.inf, d)
        try:
            want = math.ldexp(d, e)
        except OverflowError:
            want = math.copysign(math.inf, d)
        got = nt.nt_ldexp_rn(d, e)
        assert got == want or (math.isinf(got) and math.isinf(want)), (d, e, got, want)
        assert math.copysign(1, got) == math.copysign(1, want)


def _exact_round(v: int, e: int) -> float:
    """ExactValue::to_double (oracle.cpp:157-180) in Python big ints."""
    if v == 0:
        return 0.0
    neg = v < 0
    mag = -v if neg else v
    nb = mag.bit_length()
    if nb > 55:
        drop = nb - 55
        sticky = mag & ((1 << drop) - 1) != 0
        mag >>= drop
        e += drop
        if sticky and mag % 2 == 0:
            mag += 1
    try:
        r = math.ldexp(float(mag), e)
    except OverflowError:
        r = math.inf
    return -r if neg else r


def test_accumulate_and_round_against_bigints(nt):
    rng = np.random.default_rng(2)
    for trial in range(3000):
        n = int(rng.integers(1, 20))
        s = rng.integers(-2**31, 2**31, size=n, dtype=np.int64).astype(np.int32)
        if trial % 5 == 0:  # heavy cancellation
            s[1::2] = -s[::2][: len(s[1::2])]
        t = int(rng.integers(2, 8))
        shift = np.array([int(rng.integers(0, 14)) * t for _ in range(n)], dtype=np.int32)
        e = int(rng.integers(-1150, 900))
        v = sum(int(a) << int(b) for a, b in zip(s, shift))
        words = 2 if v.bit_length() < 126 and max(shift) + 33 < 127 else 3
        if max(shift) + 33 + 5 >= 64 * words:
            words = 6
        got = nt.nt_accumulate_round(words, n, s.ctypes.data, shift.ctypes.data, e)
        want = _exact_round(v, e)
        assert got == want or (math.isinf(got) and math.isinf(want)), (trial, v, e, got, want)
        out = np.zeros(6, dtype=np.uint64)
        nt.nt_accumulate_words(n, s.ctypes.data, shift.ctypes.data, out.ctypes.data)
        as_int = sum(int(w) << (64 * i) for i, w in enumerate(out))
        if as_int >> 383:
            as_int -= 1 << 384
        assert as_int == v


def test_round_words_matches_oracle(nt, po):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        n = int(rng.integers(1, 6))
        s = rng.integers(-2**31, 2**31, size=n, dtype=np.int64).astype(np.int32)
        shift = np.sort(rng.integers(0, 90, size=n)).astype(np.int32)
        e = int(rng.integers(-1100, 800))
        words = np.zeros(4, dtype=np.uint64)
        v = sum(int(a) << int(b) for a, b in zip(s, shift)) % (1 << 256)
        for i in range(4):
            words[i] = (v >> (64 * i)) & ((1 << 64) - 1)
        want = po.port().ozo_round_words(words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), 4, e)
        got = nt.nt_accumulate_round(3, n, s.ctypes.data, shift.ctypes.data, e)
        assert got == want or (math.isinf(got) and math.isinf(want))


@pytest.mark.parametrize("mode", [0, 1])
def test_slice_fields_match_oracle(nt, po, mode):
    rng = np.random.default_rng(4 + mode)
    for width, count in [(7, 12), (7, 3), (3, 20), (5, 9), (2, 6)]:
        x = np.ldexp(1.0 + rng.random((6, 40)), rng.integers(-30, 30, size=(6, 40)))
        x *= np.where(rng.random((6, 40)) < 0.5, -1.0, 1.0)
        x[0, :5] = 0.0
        sc, sl = po.port_split(x, 0, width, count, mode)
        out = np.zeros(count, dtype=np.int64)
        for i in range(6):
            for j in range(40):
                nt.nt_slices(x[i, j], int(sc[i]), width, count, mode, out.ctypes.data)
                assert np.array_equal(out, sl[:, i, j]), (i, j)


def test_round_i128_matches_bigints(nt):
    nt.nt_round_i128.restype = ctypes.c_double
    nt.nt_round_i128.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_long]
    rng = np.random.default_rng(6)
    for trial in range(20000):
        bits = int(rng.integers(1, 127))
        v = int(rng.integers(0, 2**62)) << max(0, bits - 62)
        v |= int(rng.integers(0, 2**20)) if trial % 3 else 0
        v &= (1 << 126) - 1
        if trial % 2:
            v = -v
        e = int(rng.integers(-1250, 950))
        u = v % (1 << 128)
        got = nt.nt_round_i128(u & ((1 << 64) - 1), u >> 64, e)
        want = _exact_round(v, e)
        assert got == want or (math.isinf(got) and math.isinf(want)), (v, e, got, want)


def test_round_hilo_fast_path_matches_exact(nt):
    """round_hilo (two exact conversions + one IEEE add, the combine's
    common path) equals ExactValue::to_double on random, tie-heavy and
    boundary 128-bit values (|hi| around 2..4, sticky-only low words,
    exact midpoints)."""
    nt.nt_round_hilo.restype = ctypes.c_double
    nt.nt_round_hilo.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_long]
    rng = np.random.default_rng(7)
    cases = []
    for trial in range(40000):
        kind = trial % 5
        if kind == 0:
            bits = int(rng.integers(1, 120))
            v = int(rng.integers(0, 2**62)) << max(0, bits - 62)
        elif kind == 1:  # near the fast-path boundary |v| ~ 2^64 .. 2^67
            v = int(rng.integers(2**31, 2**35)) << 32 | int(rng.integers(0, 2**32))
        elif kind == 2:  # exact ties at 53 bits: top 54 bits then zeros (+ optional sticky)
            nb = int(rng.integers(66, 118))
            top = int(rng.integers(2**53, 2**54)) | 1
            v = top << (nb - 54)
            if trial % 10 == 2:
                v += 1
        elif kind == 3:  # long carry chains in the low word
            nb = int(rng.integers(66, 118))
            v = (int(rng.integers(1, 2**20)) << (nb - 20)) - int(rng.integers(0, 2**12))
        else:  # sticky bits only below bit 11 of the low word
            v = (int(rng.integers(2**40, 2**53)) << 64) + int(rng.integers(0, 2**11))
        if trial % 2:
            v = -v
        e = int(rng.integers(-1100, 950)) if trial % 7 == 0 else int(rng.integers(-300, 100))
        cases.append((v, e))
    for v, e in cases + [(2**65, -100), (-(2**65), -100), (3 * 2**64, 5), (-(3 * 2**64) + 1, 5),
                         (2**64 + 1, 0), (-(2**64) - 1, 0), (2**116 + 2**63, -1033),
                         (2**116 - 1, 900)]:
        u = v % (1 << 128)
        got = nt.nt_round_hilo(u & ((1 << 64) - 1), u >> 64, e)
        want = _exact_round(v, e)
        assert got == want or (math.isinf(got) and math.isinf(want)), (v, e, got, want)
        assert math.copysign(1, got) == math.copysign(1, want) or want == 0, (v, e)


def test_round_w3_matches_exact(nt):
    """round_w3 (192-bit values: 128-bit path, two-term fast path, generic
    W-word path) equals ExactValue::to_double on random, boundary and tie
    cases."""
    nt.nt_round_w3.restype = ctypes.c_double
    nt.nt_round_w3.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_long]
    rng = np.random.default_rng(8)
    cases = []
    for trial in range(30000):
        kind = trial % 4
        nb = int(rng.integers(1, 180))
        if kind == 0:
            v = (int(rng.integers(0, 2**62)) << max(0, nb - 62)) | int(rng.integers(0, 2**30))
        elif kind == 1:  # around 2^128 .. 2^133 (the fast-path boundary)
            v = (int(rng.integers(1, 2**5)) << 128) + (int(rng.integers(0, 2**62)) << 64) + \
                int(rng.integers(0, 2**62))
        elif kind == 2:  # exact ties at 53 bits
            nb = int(rng.integers(131, 178))
            v = (int(rng.integers(2**53, 2**54)) | 1) << (nb - 54)
            if trial % 8 == 2:
                v += 1
        else:  # sticky bit only in the lowest word
            v = (int(rng.integers(2**10, 2**40)) << 128) + int(rng.integers(0, 3))
        v &= (1 << 190) - 1
        if trial % 2:
            v = -v
        e = int(rng.integers(-1150, 900)) if trial % 6 == 0 else int(rng.integers(-300, 60))
        cases.append((v, e))
    for v, e in cases:
        u = v % (1 << 192)
        got = nt.nt_round_w3(u & (2**64 - 1), (u >> 64) & (2**64 - 1), u >> 128, e)
        want = _exact_round(v, e)
        assert got == want or (math.isinf(got) and math.isinf(want)), (v, e, got, want)

"""Pins the C restatement (oracle/ozoracle.c) against the reference's golden
vectors (proj/tests/*_test.cpp) and against the unmodified reference compiled
from its own sources (oracle/_ref).  CPU only."""
import itertools

import numpy as np
import pytest

from helpers import bits_equal, random_matrix, uniform


# ------------------------------------------------------------ golden vectors

def test_worked_example_golden(po):
    # slicing_test.cpp:73-99 / acceptance_test.cpp:64-100 (t = 3)
    a = np.array([[1.5625, 8.0, -3.6875]])
    b = np.array([[1.3828125], [-7.625], [3.625]])
    sc, sl = po.port_split(a, 0, 3, 4)
    assert sc.tolist() == [4]
    assert sl[:, 0, :].tolist() == [[0, 4, -1], [6, 0, -6], [2, 0, -6], [0, 0, 0]]
    scb, slb = po.port_split(b, 1, 3, 4)
    assert scb.tolist() == [3]
    assert slb[:, :, 0].tolist() == [[1, -7, 3], [3, -5, 5], [0, 0, 0], [4, 0, 0]]
    # mma_sim_test.cpp:99-109
    want = {(1, 1): -31, (1, 2): -25, (2, 1): -12, (1, 3): 0, (2, 2): -12, (3, 1): -16,
            (1, 4): 0, (2, 3): 0, (3, 2): -24, (4, 1): 0}
    for (l, h), v in want.items():
        assert po.port_integer_gemm(sl[l - 1], slb[h - 1], 3, 31)[0, 0] == v
    # scheme_test.cpp:211-235
    full = po.port_multiply_exact(a, b, 4, 4, schedule=0, width=3)
    red = po.port_multiply_exact(a, b, 4, 4, schedule=1, width=3)
    assert full[0, 0] == -72.20654296875
    assert red[0, 0] == -72.21875


def test_unit_column_golden(po):
    # slicing_test.cpp:109-117: [1] -> scale 2^1, slice 4 (t = 3)
    sc, sl = po.port_split(np.array([[1.0]]), 1, 3, 2)
    assert sc.tolist() == [1] and sl[:, 0, 0].tolist() == [4, 0]


def test_plan_golden(po):
    # scheme_test.cpp:95-102, 104-111
    assert po.port_plan_levels(53, 7, 31, 8) == [(0, 3), (4, 6), (7, 7)]
    assert po.port_plan_levels(53, 7, 31, 1) == [(0, 0)]
    assert po.port_plan_levels(32, 7, 31, 5) == [(d, d) for d in range(5)]
    # scheme_test.cpp:56-78 (chi closed form vs enumeration)
    for sa, sb in itertools.product(range(1, 33), repeat=2):
        enum = sum(1 for l in range(1, sa + 1) for h in range(1, sb + 1)
                   if l + h <= max(sa, sb) + 1)
        assert po.port().ozo_chi(sa, sb) == enum
    # scheme_test.cpp:80-93
    assert po.port().ozo_spare_carries(1, 1, 7) == 127
    assert po.port().ozo_spare_carries(1, 255, 7) == 0
    # mma_sim_test.cpp:88-92 (capacity constants via the width rule)
    assert po.port().ozo_optimal_slice_width(7, 31, 65536) == 7


def test_select_slices_golden(po):
    # analysis_test.cpp:164-169
    s = po.port_select_slices(2.0, 2.0, 7, 2.0 ** -53, 24)
    assert (s["slices_a"], s["slices_b"], s["products"]) == (8, 8, 36)


def test_generator_golden(po):
    # generators_test.cpp:61-67: FNV-1a over the bit patterns of the first draws
    # is pinned against the reference generator in test_generators_match_reference;
    # here: determinism and range.
    x = po.port_random_uniform(7, 9, 5, -0.5, 0.5)
    assert np.array_equal(x, po.port_random_uniform(7, 9, 5, -0.5, 0.5))
    assert x.min() >= -0.5 and x.max() < 0.5


# ------------------------------------------------ restatement vs reference

@pytest.mark.parametrize("mode", [0, 1])
def test_split_matches_reference(po, ref, mode):
    rng = np.random.default_rng(11 + mode)
    for exps, zf in [((-4, 4), 0.0), ((-60, 60), 0.2), ((-1074, -1040), 0.0), ((1000, 1023), 0.1)]:
        x = random_matrix(9, 23, rng, *exps, zero_frac=zf)
        for width, count in [(7, 5), (3, 9), (2, 4), (11, 7), (62, 2)]:
            for orient in (0, 1):
                assert all(np.array_equal(p, q) for p, q in
                           zip(po.port_split(x, orient, width, count, mode),
                               ref.ref_split(x, orient, width, count, mode)))


def test_integer_gemm_matches_reference(po, ref):
    rng = np.random.default_rng(3)
    x = rng.integers(-128, 128, size=(7, 33))
    y = rng.integers(-128, 128, size=(33, 5))
    assert np.array_equal(po.port_integer_gemm(x, y), ref.ref_integer_gemm(x, y))
    with pytest.raises(po.RefError) as e:
        po.port_integer_gemm(np.full((2, 64), 127), np.full((64, 2), 127), 7, 19)
    assert e.value.code == 5


@pytest.mark.parametrize("case", range(6))
def test_multiply_exact_matches_reference(po, ref, case):
    rng = np.random.default_rng(100 + case)
    m, k, n = [(5, 9, 4), (17, 40, 23), (8, 130, 6), (33, 64, 31), (3, 5, 7), (12, 257, 9)][case]
    if case % 2:
        a, b = uniform(m, k, rng), uniform(k, n, rng)
    else:
        a = random_matrix(m, k, rng, -25, 25, 0.05)
        b = random_matrix(k, n, rng, -25, 25, 0.05)
    for (sa, sb), sched, mode in itertools.product([(1, 1), (4, 4), (3, 7), (9, 8)], (0, 1), (0, 1)):
        got = po.port_multiply_exact(a, b, sa, sb, schedule=sched, mode=mode)
        want, _ = ref.ref_multiply(a, b, sa, sb, sched, 2, mode)
        assert bits_equal(got, want), (sa, sb, sched, mode)


def test_multiply_exact_badly_scaled(po, ref):
    a, b = po.port_gen_kappa_d(48, 2.0 ** 60, 7, True)
    wa, wb = ref.ref_gen_kappa_d(48, 2.0 ** 60, 7, True)
    assert bits_equal(a, wa) and bits_equal(b, wb)
    for sa, sb in [(8, 8), (16, 17)]:
        got = po.port_multiply_exact(a, b, sa, sb)
        want, _ = ref.ref_multiply(a, b, sa, sb)
        assert bits_equal(got, want)


def test_diag_sum_limit_matches_reference(po, ref):
    rng = np.random.default_rng(14)
    a = random_matrix(6, 8, rng, -6, 6)
    b = random_matrix(8, 6, rng, -6, 6)
    got = po.port_multiply_exact(a, b, 5, 5, schedule=1, diag_sum_limit=5)
    want, _ = ref.ref_multiply(a, b, 5, 5, 1, 2, 0, 53, 5)
    assert bits_equal(got, want)


def test_plan_and_estimator_match_reference(po, ref):
    for p, t, tu, d in itertools.product((53, 40, 33), (2, 3, 7, 11), (14, 18, 25, 31),
                                         (1, 2, 5, 8, 20, 60)):
        if tu >= p:
            continue
        assert po.port_plan_levels(p, t, tu, d) == ref.ref_plan_levels(p, t, tu, d)
    for ka, kb, t, target, sched, strat in itertools.product(
            (2.0, 3.5, 2.0 ** 20, 2.0 ** 62), (2.0, 1e9), (7, 5), (None, 1e-15, 1e-30),
            (0, 1), (0, 1, 2)):
        got = po.port_select_slices(ka, kb, t, 2.0 ** -53, 24, target, sched, strat, 2 * t + 13)
        want = ref.ref_select_slices(ka, kb, t, 2.0 ** -53, 24, target, sched, strat, 2 * t + 13)
        assert got == want


def test_scaling_profile_matches_reference(po, ref):
    rng = np.random.default_rng(8)
    a = random_matrix(20, 30, rng, -40, 40, 0.2)
    b = random_matrix(30, 10, rng, -40, 40, 0.2)
    a[4] = 0.0
    b[:, 2] = 0.0
    assert po.port_scaling_profile(a, b) == ref.ref_scaling_profile(a, b)


def test_generators_match_reference(po, ref):
    assert bits_equal(po.port_random_uniform(64, 33, 1, -0.5, 0.5),
                      ref.ref_random_uniform(64, 33, 1, -0.5, 0.5))
    assert bits_equal(po.port_random_uniform(5, 5, 2), ref.ref_random_uniform(5, 5, 2))

"""Seeded random sweep over the multiply() surface against the reference
(scheme.cpp:219-361, compiled in place): shapes from 1 to a few hundred
(ragged against every tile / k-block size), slice counts 1..12, both
schedules, all three accumulation strategies, both slicing modes, narrow and
wide exponent ranges with zeros, host and device-pointer entry points.  C
must match bit for bit and the Diagnostics exactly.  (Scaled products that
underflow are excluded: DESIGN.md §2 covers that regime separately.)"""
import numpy as np
import pytest

from helpers import bits_equal, mismatch_report, random_matrix

pytestmark = pytest.mark.gpu

CASES = 96


def _case(i):
    rng = np.random.default_rng(1000 + i)
    m = int(rng.integers(1, 260))
    n = int(rng.integers(1, 260))
    k = int(rng.integers(1, 700))
    sa = int(rng.integers(1, 13))
    sb = int(rng.integers(1, 13))
    schedule = int(rng.integers(0, 2))
    strategy = int(rng.choice([2, 2, 1, 0]))
    mode = int(rng.integers(0, 2))
    span = int(rng.choice([2, 8, 24]))
    zero = float(rng.choice([0.0, 0.0, 0.2]))
    a = random_matrix(m, k, rng, -span, span, zero)
    b = random_matrix(k, n, rng, -span, span, zero)
    device = bool(rng.integers(0, 2))
    return m, n, k, sa, sb, schedule, strategy, mode, a, b, device


@pytest.mark.parametrize("i", range(CASES))
def test_random_multiply_matches_reference(oz, ref, i):
    m, n, k, sa, sb, schedule, strategy, mode, a, b, device = _case(i)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, sa, sb, schedule=oz.ScheduleKind(schedule),
                        strategy=oz.Accumulation(strategy), mode=oz.SliceMode(mode))
    want, wdiag = ref.ref_multiply(a, b, sa, sb, schedule, strategy, mode)
    if device:
        import torch
        dev = torch.device("cuda:0")
        da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
        dc = torch.empty((m, n), dtype=torch.float64, device=dev)
        s = torch.cuda.Stream(device=dev)
        d = oz.multiply_device(m, n, k, da.data_ptr(), k, db.data_ptr(), n, dc.data_ptr(), n, cfg,
                               plan, stream=s.cuda_stream)
        s.synchronize()
        got = dc.cpu().numpy()
    else:
        r = oz.multiply(a, b, cfg, plan)
        got, d = r.c, r.diagnostics
    what = (m, n, k, sa, sb, schedule, strategy, mode, "device" if device else "host")
    assert bits_equal(got, want), (what, mismatch_report(got, want))
    # every Diagnostics field; realized_psi (the sequential strategies'
    # inexact TwoSum count, read back from the GPU) only on the host path --
    # the device-pointer call returns before the GPU has run
    got_d = [d.products, d.integer_adds, d.float_adds, d.flushes, d.realized_psi, d.planned_psi,
             d.width, d.acc_bits_used]
    want_d = wdiag.tolist()
    if device:
        got_d[4] = want_d[4] = 0
    assert got_d == want_d, what


@pytest.mark.parametrize("i", range(24))
def test_random_axpby_matches_reference(oz, ref, i):
    """multiply_axpby (scheme.cpp:363-372): D = alpha AB + beta C with the
    reference's two roundings, over random shapes, slices and scalars."""
    rng = np.random.default_rng(5000 + i)
    m, n, k = (int(rng.integers(1, 200)) for _ in range(3))
    sa, sb = int(rng.integers(1, 10)), int(rng.integers(1, 10))
    a = random_matrix(m, k, rng, -10, 10, 0.1)
    b = random_matrix(k, n, rng, -10, 10, 0.1)
    c = random_matrix(m, n, rng, -10, 10, 0.1)
    alpha, beta = (float(x) for x in rng.choice([1.0, -1.0, 0.5, 3.25, 0.0, -2.0e-3], 2))
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, sa, sb)
    got = oz.multiply_axpby(alpha, a, b, beta, c, cfg, plan).c
    want = ref.ref_multiply_axpby(alpha, a, b, beta, c, sa, sb)
    assert bits_equal(got, want), ((m, n, k, sa, sb, alpha, beta), mismatch_report(got, want))


@pytest.mark.parametrize("i", range(24))
def test_random_split_and_estimator_match_reference(oz, ref, i):
    """split_rows / split_cols (slicing.cpp:67-132) bit-exact at random widths,
    counts and modes, and the estimator's kappa scan + select_slices
    (analysis.cpp:25-68, 142-207) on the same random operands."""
    rng = np.random.default_rng(7000 + i)
    rows, cols = int(rng.integers(1, 120)), int(rng.integers(1, 120))
    width = int(rng.integers(1, 8))
    mode = int(rng.integers(0, 2)) if width >= 2 else 0
    count = int(rng.integers(1, 14))
    x = random_matrix(rows, cols, rng, -30, 30, 0.15)
    for orientation in (0, 1):
        sm = (oz.split_rows if orientation == 0 else oz.split_cols)(x, width, count,
                                                                     oz.SliceMode(mode))
        wsc, wsl = ref.ref_split(x, orientation, width, count, mode)
        assert np.array_equal(sm.scale_exponents, wsc), (orientation, width, count, mode)
        assert np.array_equal(sm.slices, wsl), (orientation, width, count, mode)
    k = cols
    b = random_matrix(k, int(rng.integers(1, 90)), rng, -25, 25, 0.1)
    prof = oz.scaling_profile(x, b)
    ka, kb, za, zb = ref.ref_scaling_profile(x, b)
    assert (prof.kappa_a, prof.kappa_b, prof.a_has_zero_block, prof.b_has_zero_block) == \
        (ka, kb, za, zb)
    target = float(rng.choice([1e-8, 1e-12, 1e-15]))
    want = ref.ref_select_slices(ka, kb, 7, 2.0 ** -53, 24, target=target)
    if want.get("infeasible"):
        with pytest.raises(oz.SelectionInfeasible):
            oz.select_slices(ka, kb, 7, 2.0 ** -53, 24, oz.SelectOptions(target=target))
        return
    got = oz.select_slices(ka, kb, 7, 2.0 ** -53, 24, oz.SelectOptions(target=target))
    assert (got.slices_a, got.slices_b, got.products) == \
        (want["slices_a"], want["slices_b"], want["products"])
    assert got.lhs == want["lhs"] and got.target == want["target"]

"""The product library's host-side plan / estimator logic (no GPU needed)
against the compiled reference, plus the reference's error contracts."""
import itertools

import pytest


def test_make_plan_matches_reference(oz, ref):
    cfg = oz.MmaConfig.int8_int32()
    for k, (sa, sb), sched, strat, mode, prec in itertools.product(
            (1, 2, 3, 100, 1024, 8192, 16384, 32768, 65536),
            [(1, 1), (4, 4), (12, 12), (13, 12), (16, 17), (3, 9)], (0, 1), (0, 1, 2), (0, 1),
            (53, 40)):
        try:
            want = ref.ref_make_plan(k, sa, sb, sched, strat, mode, prec)
        except ref.RefError as e:
            with pytest.raises(oz.OzmulError) as got:
                oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind(sched), oz.Accumulation(strat),
                             oz.SliceMode(mode), prec)
            assert got.value.code == e.code
            continue
        p = oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind(sched), oz.Accumulation(strat),
                         oz.SliceMode(mode), prec)
        assert (p.width, p.acc_bits_used, p.psi, p.levels) == \
            (want["width"], want["acc_bits_used"], want["psi"], want["levels"])


def test_plan_functions_match_reference(oz, ref):
    for sa, sb in itertools.product(range(1, 40), repeat=2):
        assert oz.chi(sa, sb) == ref.ref().ozref_chi(sa, sb)
    for p, t, tu, d in itertools.product((53, 40, 33), (2, 3, 7, 11), (14, 18, 25, 31),
                                         (1, 2, 5, 8, 20, 60)):
        if tu >= p:
            continue
        assert oz.plan_levels(p, t, tu, d)[0] == ref.ref_plan_levels(p, t, tu, d)
    assert oz.plan_levels(53, 7, 31, 8) == ([(0, 3), (4, 6), (7, 7)], 2)


def test_reference_constants(oz):
    cfg = oz.MmaConfig.int8_int32()
    # mma_sim_test.cpp:88-92, scheme_test.cpp:195-200
    assert oz.max_inner_dim(cfg) == 65536
    assert oz.max_inner_dim(oz.MmaConfig(3, 31)) == 16777216
    assert oz.diagonal_flush_threshold(cfg, 7, 1024) == 128
    assert oz.diagonal_flush_threshold(cfg, 1, 2) == 1 << 28
    assert oz.optimal_slice_width(cfg, 65536) == 7
    assert oz.spare_carries(1, 1, 7) == 127 and oz.spare_carries(1, 255, 7) == 0


def test_select_slices_matches_reference(oz, ref):
    for ka, kb, t, target, sched, strat, smax in itertools.product(
            (2.0, 3.5, 2.0 ** 20, 2.0 ** 34, 2.0 ** 62), (2.0, 1e9), (7, 5), (None, 1e-15, 1e-30),
            (0, 1), (0, 1, 2), (24, 8)):
        want = ref.ref_select_slices(ka, kb, t, 2.0 ** -53, smax, target, sched, strat, 2 * t + 13)
        opts = oz.SelectOptions(target=target, schedule=oz.ScheduleKind(sched),
                                strategy=oz.Accumulation(strat), acc_bits_used=2 * t + 13)
        if want.get("infeasible"):
            with pytest.raises(oz.SelectionInfeasible) as e:
                oz.select_slices(ka, kb, t, 2.0 ** -53, smax, opts)
            assert (e.value.gap, e.value.best_lhs, e.value.target) == \
                (want["gap"], want["lhs"], want["target"])
            continue
        got = oz.select_slices(ka, kb, t, 2.0 ** -53, smax, opts)
        assert (got.slices_a, got.slices_b, got.lhs, got.target, got.products) == \
            (want["slices_a"], want["slices_b"], want["lhs"], want["target"], want["products"])
    # analysis_test.cpp:164-169
    s = oz.select_slices(2.0, 2.0, 7, 2.0 ** -53, 24)
    assert (s.slices_a, s.slices_b, s.products) == (8, 8, 36)


def test_error_contracts(oz):
    cfg = oz.MmaConfig.int8_int32()
    with pytest.raises(oz.InvalidArgument):
        oz.chi(0, 3)
    with pytest.raises(oz.InvalidArgument):
        oz.make_plan(cfg, 16, 0, 2)
    with pytest.raises(oz.InvalidArgument):
        oz.spare_carries(0, 1, 7)
    with pytest.raises(oz.InvalidArgument):
        oz.select_slices(-1.0, 2.0, 7, 2.0 ** -53, 24)
    with pytest.raises(oz.InvalidArgument):
        oz.make_plan(oz.MmaConfig(7, 63), 16, 2, 2)  # MmaConfig::validate
    with pytest.raises(oz.DomainError):
        oz.optimal_slice_width(oz.MmaConfig(7, 31), 1 << 40)
    with pytest.raises(oz.SelectionInfeasible):
        oz.select_slices(1e300, 1e300, 7, 2.0 ** -53, 2, oz.SelectOptions(target=1e-30))


def test_generators_match_reference(oz, ref):
    from helpers import bits_equal
    assert bits_equal(oz.random_uniform(40, 37, 1, -0.5, 0.5),
                      ref.ref_random_uniform(40, 37, 1, -0.5, 0.5))
    a, b = oz.gen_kappa_d(33, 2.0 ** 60, 7, True)
    wa, wb = ref.ref_gen_kappa_d(33, 2.0 ** 60, 7, True)
    assert bits_equal(a, wa) and bits_equal(b, wb)

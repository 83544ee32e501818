"""GPU parity: the CUDA path through the C-ABI against the compiled reference
(oracle/_ref) and the C restatement, bit-exact (slices, pair products, the
levelled-exact C, and the sequential strategies in matched order)."""
import itertools

import numpy as np
import pytest

from helpers import bits_equal, mismatch_report, random_matrix, ref_full, uniform

pytestmark = pytest.mark.gpu

STRATS = (0, 1, 2)


def _diag_tuple(d):
    return (d.products, d.integer_adds, d.float_adds, d.flushes, d.realized_psi, d.planned_psi,
            d.width, d.acc_bits_used)


# ---------------------------------------------------------------- slicing

@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (17, 130), (64, 257), (9, 1000)])
@pytest.mark.parametrize("mode", [0, 1])
def test_split_matches_reference(oz, ref, shape, mode):
    rng = np.random.default_rng(hash((shape, mode)) % 2**32)
    for exps, zf in [((-4, 4), 0.0), ((-40, 40), 0.1), ((-1074, -1000), 0.0), ((1000, 1023), 0.2)]:
        x = random_matrix(*shape, rng, *exps, zero_frac=zf)
        for width, count in [(7, 4), (7, 9), (3, 5), (5, 17), (2, 3)]:
            sa = oz.split_rows(x, width, count, oz.SliceMode(mode))
            wsc, wsl = ref.ref_split(x, 0, width, count, mode)
            assert np.array_equal(sa.scale_exponents, wsc)
            assert np.array_equal(sa.slices, wsl), (exps, width, count)
            sb = oz.split_cols(x, width, count, oz.SliceMode(mode))
            wsc, wsl = ref.ref_split(x, 1, width, count, mode)
            assert np.array_equal(sb.scale_exponents, wsc)
            assert np.array_equal(sb.slices, wsl), (exps, width, count)


def test_split_wide_widths_and_errors(oz, ref):
    rng = np.random.default_rng(5)
    x = random_matrix(7, 11, rng, -30, 30, zero_frac=0.1)
    for width, count in [(20, 3), (62, 2), (11, 6)]:
        for mode in (0, 1):
            s = oz.split_rows(x, width, count, oz.SliceMode(mode))
            wsc, wsl = ref.ref_split(x, 0, width, count, mode)
            assert np.array_equal(s.slices, wsl) and np.array_equal(s.scale_exponents, wsc)
    bad = x.copy()
    bad[2, 3] = np.inf
    with pytest.raises(oz.InvalidArgument):
        oz.split_rows(bad, 7, 2)
    negz = x.copy()
    negz[0, 0] = -0.0  # split accepts negative zeros (only multiply rejects them)
    s = oz.split_rows(negz, 7, 2)
    assert s.slices[:, 0, 0].tolist() == [0, 0]
    with pytest.raises(oz.InvalidArgument):
        oz.split_rows(x, 0, 2)
    with pytest.raises(oz.InvalidArgument):
        oz.split_rows(x, 7, 0)


def test_golden_worked_example_slices(oz):
    # proj/tests/slicing_test.cpp:73-99, acceptance_test.cpp:64-100
    a = np.array([[1.5625, 8.0, -3.6875]])
    b = np.array([[1.3828125], [-7.625], [3.625]])
    sa = oz.split_rows(a, 3, 4)
    sb = oz.split_cols(b, 3, 4)
    assert sa.scale_exponents.tolist() == [4] and sb.scale_exponents.tolist() == [3]
    assert sa.slices[:, 0, :].tolist() == [[0, 4, -1], [6, 0, -6], [2, 0, -6], [0, 0, 0]]
    assert sb.slices[:, :, 0].tolist() == [[1, -7, 3], [3, -5, 5], [0, 0, 0], [4, 0, 0]]
    cfg = oz.MmaConfig(3, 31)
    want = {(1, 1): -31, (1, 2): -25, (2, 1): -12, (1, 3): 0, (2, 2): -12, (3, 1): -16,
            (1, 4): 0, (2, 3): 0, (3, 2): -24, (4, 1): 0}
    for (l, h), v in want.items():
        e = oz.integer_gemm(sa.slices[l - 1], sb.slices[h - 1], cfg)
        assert e[0, 0] == v
    full = oz.make_plan(cfg, 3, 4, 4, oz.ScheduleKind.FULL)
    assert oz.multiply(a, b, cfg, full).c[0, 0] == -72.20654296875
    red = oz.make_plan(cfg, 3, 4, 4, oz.ScheduleKind.REDUCED)
    r = oz.multiply(a, b, cfg, red)
    assert r.c[0, 0] == -72.21875
    assert r.diagnostics.products == oz.chi(4, 4)


# --------------------------------------------------------- pair products

@pytest.mark.parametrize("mkn", [(1, 1, 1), (5, 3, 7), (128, 128, 256), (130, 300, 257),
                                 (257, 1024, 129)])
def test_integer_gemm_tensor_path(oz, ref, mkn):
    m, k, n = mkn
    rng = np.random.default_rng(m * 1000 + n)
    x = rng.integers(-128, 128, size=(m, k))
    y = rng.integers(-128, 128, size=(k, n))
    cfg = oz.MmaConfig.int8_int32()
    got = oz.integer_gemm(x, y, cfg)
    assert np.array_equal(got, ref.ref_integer_gemm(x, y))
    c = rng.integers(-1000, 1000, size=(m, n))
    got_c = oz.integer_gemm(x, y, cfg, c)
    assert np.array_equal(got_c, ref.ref_integer_gemm(x, y) + c)


def test_integer_gemm_overflow_matches_reference(oz, ref):
    rng = np.random.default_rng(3)
    x = rng.integers(120, 128, size=(4, 64))
    y = rng.integers(120, 128, size=(64, 5))
    cfg = oz.MmaConfig(7, 19)  # 64 * 127^2 exceeds I_19
    with pytest.raises(ref.RefError) as want:
        ref.ref_integer_gemm(x, y, 7, 19)
    assert want.value.code == 5
    with pytest.raises(oz.MmaOverflowError) as got:
        oz.integer_gemm(x, y, cfg)
    assert str(got.value) == want.value.msg
    with pytest.raises(oz.DomainError):
        oz.integer_gemm(np.full((2, 2), 200), y[:2], cfg)


# ---------------------------------------------------------------- multiply

SHAPES = [(1, 1, 1), (5, 7, 3), (33, 100, 17), (129, 257, 130), (200, 64, 300)]


@pytest.mark.parametrize("mkn", SHAPES)
def test_multiply_levelled_matches_reference(oz, ref, mkn):
    m, k, n = mkn
    rng = np.random.default_rng(sum(mkn))
    cfg = oz.MmaConfig.int8_int32()
    inputs = [(uniform(m, k, rng), uniform(k, n, rng)),
              (random_matrix(m, k, rng, -20, 20, 0.05), random_matrix(k, n, rng, -20, 20, 0.05))]
    for (a, b), (sa, sb), sched, mode in itertools.product(
            inputs, [(1, 1), (4, 4), (3, 7), (8, 8), (13, 12)], (0, 1), (0, 1)):
        plan = oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind(sched), oz.Accumulation(2),
                            oz.SliceMode(mode))
        got = oz.multiply(a, b, cfg, plan)
        want, wd = ref.ref_multiply(a, b, sa, sb, sched, 2, mode)
        assert bits_equal(got.c, want), (sa, sb, sched, mode, mismatch_report(got.c, want))
        assert _diag_tuple(got.diagnostics) == tuple(wd.tolist())


@pytest.mark.parametrize("strategy", [0, 1])
def test_multiply_sequential_strategies_match_reference(oz, ref, strategy):
    rng = np.random.default_rng(40 + strategy)
    cfg = oz.MmaConfig.int8_int32()
    for (m, k, n) in [(6, 9, 5), (64, 300, 70), (130, 129, 33)]:
        a = random_matrix(m, k, rng, -12, 12, 0.05)
        b = random_matrix(k, n, rng, -12, 12, 0.05)
        for (sa, sb), sched, mode in itertools.product([(3, 3), (6, 6), (5, 9)], (0, 1), (0, 1)):
            plan = oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind(sched),
                                oz.Accumulation(strategy), oz.SliceMode(mode))
            got = oz.multiply(a, b, cfg, plan)
            want, wd = ref.ref_multiply(a, b, sa, sb, sched, strategy, mode)
            assert bits_equal(got.c, want), (m, k, n, sa, sb, sched, mode,
                                              mismatch_report(got.c, want))
            assert _diag_tuple(got.diagnostics) == tuple(wd.tolist())


def test_multiply_error_free_at_exact_slice_counts(oz, ref):
    # acceptance criterion 2 (acceptance_test.cpp:105-133), fewer seeds
    rng = np.random.default_rng(20250809)
    cfg = oz.MmaConfig.int8_int32()
    for _ in range(25):
        m, k, n = (int(v) for v in rng.integers(1, 33, size=3))
        a = random_matrix(m, k, rng, -40, 40)
        b = random_matrix(k, n, rng, -40, 40)
        t = oz.optimal_slice_width(cfg, k)
        sa = ref.ref_min_exact_slices(a, 0, t)
        sb = ref.ref_min_exact_slices(b, 1, t)
        plan = oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind.FULL)
        got = oz.multiply(a, b, cfg, plan).c
        assert bits_equal(got, ref.ref_exact_gemm(a, b))


def test_multiply_input_errors(oz):
    cfg = oz.MmaConfig.int8_int32()
    a = np.ones((1, 2))
    b = np.ones((2, 1))
    plan = oz.make_plan(cfg, 2, 1, 1)
    for bad in (np.inf, np.nan, -0.0):
        aa = a.copy()
        aa[0, 1 if bad != -0.0 else 0] = bad
        with pytest.raises(oz.InvalidArgument):
            oz.multiply(aa, b, cfg, plan)
    forged = oz.make_plan(cfg, 2, 2, 2)
    forged.width = 16  # scheme_test.cpp:294-302
    with pytest.raises(oz.DomainError, match="65536"):
        oz.multiply(a, b, cfg, forged)
    with pytest.raises(oz.InvalidArgument):
        oz.multiply(np.ones((1, 0)), np.ones((0, 1)), cfg, plan)
    with pytest.raises(oz.InvalidArgument):
        oz.multiply(np.ones((2, 3)), np.ones((2, 3)), cfg, plan)


def test_multiply_axpby_matches_reference(oz, ref):
    rng = np.random.default_rng(21)
    cfg = oz.MmaConfig.int8_int32()
    a = random_matrix(40, 60, rng)
    b = random_matrix(60, 50, rng)
    c = random_matrix(40, 50, rng)
    for sa, sb, sched in [(4, 4, 0), (8, 8, 1)]:
        plan = oz.make_plan(cfg, 60, sa, sb, oz.ScheduleKind(sched))
        got = oz.multiply_axpby(-2.5, a, b, 0.5, c, cfg, plan).c
        want = ref.ref_multiply_axpby(-2.5, a, b, 0.5, c, sa, sb, sched)
        assert bits_equal(got, want)


def test_scaling_profile_matches_reference(oz, ref):
    rng = np.random.default_rng(9)
    a = random_matrix(50, 70, rng, -30, 30, 0.1)
    b = random_matrix(70, 40, rng, -30, 30, 0.1)
    a[3, :] = 0.0
    p = oz.scaling_profile(a, b)
    assert (p.kappa_a, p.kappa_b, p.a_has_zero_block, p.b_has_zero_block) == \
        ref.ref_scaling_profile(a, b)


def test_badly_scaled_kappa_d(oz, ref):
    # acceptance criterion 8 style: gen_kappa_d with rotation, bit-exact C
    a, b = oz.gen_kappa_d(96, 2.0**60, 7, True)
    wa, wb = ref.ref_gen_kappa_d(96, 2.0**60, 7, True)
    assert bits_equal(a, wa) and bits_equal(b, wb)
    cfg = oz.MmaConfig.int8_int32()
    for sa, sb in [(8, 8), (16, 17)]:
        plan = oz.make_plan(cfg, 96, sa, sb)
        got = oz.multiply(a, b, cfg, plan).c
        want, _ = ref.ref_multiply(a, b, sa, sb)
        assert bits_equal(got, want), mismatch_report(got, want)


def test_native_kernels_launched(oz):
    cfg = oz.MmaConfig.int8_int32()
    before = oz.kernel_launches()
    oz.multiply(np.ones((8, 8)), np.ones((8, 8)), cfg, oz.make_plan(cfg, 8, 2, 2))
    assert oz.kernel_launches() - before >= 3  # slicing, pair GEMM, combine


GEMM_VARIANTS = {
    "default": {},
    "final": {"OZGPU_EPILOGUE": "final", "OZGPU_CTA_PAIR": "0"},
    "fused": {"OZGPU_EPILOGUE": "fused", "OZGPU_CTA_PAIR": "0"},
    "pair_bins_lockstep": {"OZGPU_BINS": "1"},
    "pair_bins_lockstep_g1": {"OZGPU_BINS": "1", "OZGPU_SYNC_G": "1", "OZGPU_SYNC_D": "1"},
    "pair_no_lockstep": {"OZGPU_BINS": "1", "OZGPU_SYNC": "0"},
    "pair_stages3": {"OZGPU_PAIR_STAGES": "3", "OZGPU_BINS": "1"},
    "pair_n256": {"OZGPU_PAIR_N": "256", "OZGPU_BINS": "1"},
    "pair_n256_stages4": {"OZGPU_PAIR_N": "256", "OZGPU_PAIR_STAGES": "4", "OZGPU_BINS": "1"},
    "no_bins": {"OZGPU_BINS": "0"},
    "multicast_1cta": {"OZGPU_CTA_PAIR": "0"},
    "multicast_1cta_bins_lockstep": {"OZGPU_CTA_PAIR": "0", "OZGPU_BINS": "1"},
    "plain_1cta_bins": {"OZGPU_CTA_PAIR": "0", "OZGPU_MC": "0", "OZGPU_BINS": "1"},
    "horner_combine": {"OZGPU_COMBINE": "horner"},
    "plane_budget_row_blocks": {"OZGPU_PLANE_BUDGET_GB": "0.002"},
    "pair_n512_3stages_no_lockstep": {"OZGPU_PAIR_N": "512", "OZGPU_PAIR_STAGES": "3",
                                      "OZGPU_SYNC": "0"},
    "quad_clusters": {"OZGPU_QUAD": "1", "OZGPU_BINS": "1"},
    "slice_queue": {"OZGPU_SLICE_QUEUE": "1"},
    "slice_queue_small_panels": {"OZGPU_SLICE_QUEUE": "1", "OZGPU_SLICE_PANEL_MB": "1",
                                 "OZGPU_SLICE_LOOKAHEAD": "2"},
}


_VARIANT_CASES = []


def _variant_cases(ref):
    """Inputs and reference results shared by every GEMM variant (computed
    once: the reference's scalar loop dominates the test time)."""
    if not _VARIANT_CASES:
        rng = np.random.default_rng(77)
        for (m, k, n) in [(128, 256, 256), (300, 500, 700), (520, 128, 260)]:
            a = uniform(m, k, rng)
            b = random_matrix(k, n, rng, -30, 30, 0.02)
            for (sa, sb), sched in [((4, 4), 1), ((13, 12), 1), ((16, 17), 1), ((6, 7), 0)]:
                _VARIANT_CASES.append((a, b, sa, sb, sched, ref_full(ref, a, b, sa, sb, sched)))
        a = uniform(256, 384, rng)
        b = uniform(384, 512, rng)
        c = uniform(256, 512, rng)
        _VARIANT_CASES.append((a, b, c, ref.ref_multiply_axpby(1.5, a, b, -0.25, c, 7, 7)))
    return _VARIANT_CASES


@pytest.mark.parametrize("variant", sorted(GEMM_VARIANTS))
def test_gemm_variants_match_reference(oz, ref, variant, monkeypatch):
    """Every GEMM variant -- the CTA-pair (cta_group::2) kernel with 256 x 512
    (default) and 256 x 256 tiles, with and without wave lockstep and at 3-6
    stages, the B-multicast and plain
    1-CTA kernels, equal-length chunk bins on / off, the fused W-word and
    folded-combine epilogues, both exact combine kernels -- is bit-exact,
    incl. ragged tiles and 3-word exact values."""
    cases = _variant_cases(ref)
    for key, val in GEMM_VARIANTS[variant].items():
        monkeypatch.setenv(key, val)
    cfg = oz.MmaConfig.int8_int32()
    for a, b, sa, sb, sched, want in cases[:-1]:
        plan = oz.make_plan(cfg, a.shape[1], sa, sb, oz.ScheduleKind(sched))
        got = oz.multiply(a, b, cfg, plan).c
        assert bits_equal(got, want), (a.shape, b.shape, sa, sb, mismatch_report(got, want))
    # axpby through the fused epilogue
    a, b, c, want = cases[-1]
    plan = oz.make_plan(cfg, 384, 7, 7)
    got = oz.multiply_axpby(1.5, a, b, -0.25, c, cfg, plan).c
    assert bits_equal(got, want)


@pytest.mark.parametrize("k,slices", [(20000, (12, 12)), (70000, (6, 5)), (131072, (3, 3))])
def test_long_k_multi_chunk_diagonals(oz, ref, k, slices):
    """k large enough that a diagonal's int32 capacity holds fewer pairs than
    the diagonal has (cap = floor((2^31-1) / (k 127^2)): 8 at k=20000, 1 at
    k >= 65536), so diagonals split into several chunks."""
    rng = np.random.default_rng(k)
    m, n = 24, 20
    a = uniform(m, k, rng)
    b = random_matrix(k, n, rng, -3, 3, 0.01)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, *slices)
    got = oz.multiply(a, b, cfg, plan)
    blocks = [(0, 12, 0, 10), (0, 12, 10, 20), (12, 24, 0, 10), (12, 24, 10, 20)]
    want, _ = ref.ref_multiply_blocks(a, b, slices[0], slices[1], blocks, 4)
    assert bits_equal(got.c, want), mismatch_report(got.c, want)


def test_concurrent_callers_are_safe(oz, ref):
    """multiply is called from host thread pools in the reference CLI
    (main.cpp:422,486,557); results must stay bitwise deterministic."""
    import concurrent.futures as cf
    rng = np.random.default_rng(99)
    cfg = oz.MmaConfig.int8_int32()
    cases = []
    for i in range(12):
        m, k, n = (int(v) for v in rng.integers(8, 200, size=3))
        a, b = uniform(m, k, rng), uniform(k, n, rng)
        cases.append((a, b, oz.make_plan(cfg, k, 4 + i % 5, 3 + i % 4)))
    want = [oz.multiply(a, b, cfg, p).c for a, b, p in cases]
    with cf.ThreadPoolExecutor(8) as ex:
        got = list(ex.map(lambda c: oz.multiply(c[0], c[1], cfg, c[2]).c, cases * 3))
    for i, g in enumerate(got):
        assert bits_equal(g, want[i % len(cases)])


def test_large_shape_sampled_blocks(oz, ref):
    """A 2304 x 4096 x 2176 product (ragged vs the 128 x 256 tiles) with the
    estimator's slices: sampled 32 x 32 blocks equal the reference's (blocking
    is exact)."""
    m, k, n = 2304, 4096, 2176
    a = oz.random_uniform(m, k, 1, -0.5, 0.5)
    b = oz.random_uniform(k, n, 2, -0.5, 0.5)
    cfg = oz.MmaConfig.int8_int32()
    prof = oz.scaling_profile(a, b)
    t = oz.optimal_slice_width(cfg, k)
    sel = oz.select_slices(prof.kappa_a, prof.kappa_b, t, 2.0 ** -53, 24,
                           oz.SelectOptions(target=1e-15, acc_bits_used=2 * t + 12))
    plan = oz.make_plan(cfg, k, sel.slices_a, sel.slices_b)
    c = oz.multiply(a, b, cfg, plan).c
    blocks = [(r, r + 32, q, q + 32) for r, q in [(0, 0), (2272, 2144), (1000, 517), (128, 2000),
                                                  (2200, 64), (640, 1280), (1500, 1500), (32, 31)]]
    want, _ = ref.ref_multiply_blocks(a, b, sel.slices_a, sel.slices_b, blocks, 8)
    for r0, r1, c0, c1 in blocks:
        assert bits_equal(c[r0:r1, c0:c1], want[r0:r1, c0:c1]), (r0, c0)


def test_error_bound_matches_reference_and_contains(oz, ref):
    """analysis.cpp:86-131 (|A||B| on the GPU in the reference's order): the
    bound matrix equals the reference's bitwise and contains |C - exact|."""
    rng = np.random.default_rng(31)
    cfg = oz.MmaConfig.int8_int32()
    a = random_matrix(40, 90, rng, -8, 8, 0.05)
    b = random_matrix(90, 30, rng, -8, 8, 0.05)
    for sa, sb, sched in [(3, 4, 1), (5, 5, 0), (6, 3, 1)]:
        plan = oz.make_plan(cfg, 90, sa, sb, oz.ScheduleKind(sched))
        rep = oz.error_bound(a, b, plan)
        coef, bound = ref.ref_error_bound(a, b, sa, sb, sched)
        assert rep.coefficient == coef
        assert bits_equal(rep.bound, bound)
        c = oz.multiply(a, b, cfg, plan).c
        exact = ref.ref_exact_gemm(a, b)
        assert (np.abs(c - exact) <= rep.bound).all()
    assert oz.kappa(a, oz.BlockOrientation.ROWS) == ref.ref_scaling_profile(a, b)[0]


@pytest.mark.parametrize("rows,panels,last,mode,first", [
    ("4", "2", "2", "panels", "1"), ("3", "4", "3", "panels", "2"), ("8", "1", "1", "panels", "1"),
    ("4", "4", "2", "rect", "1"), ("3", "5", "2", "rect", "2"), ("4", "4", "4", "rect", "2"),
    ("5", "3", "3", "rect", "3")])
def test_blocked_host_pipeline_is_bitwise_identical(oz, rows, panels, last, mode, first, monkeypatch):
    """ozgpu_dgemm's blocked H2D / compute / D2H pipeline (row blocks, B
    column panels, a smaller first block and panel, split last block)
    returns exactly the unblocked result on a ragged shape, for several
    blockings."""
    rng = np.random.default_rng(5)
    m, k, n = 2600, 1000, 3000
    a = uniform(m, k, rng)
    b = random_matrix(k, n, rng, -20, 20, 0.01)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, 9, 8)
    monkeypatch.setenv("OZGPU_PIPE", "0")
    want = oz.multiply(a, b, cfg, plan).c
    monkeypatch.setenv("OZGPU_PIPE", "1")
    monkeypatch.setenv("OZGPU_PIPE_ROWS", rows)
    monkeypatch.setenv("OZGPU_PIPE_PANELS", panels)
    monkeypatch.setenv("OZGPU_PIPE_LAST", last)
    monkeypatch.setenv("OZGPU_PIPE_MODE", mode)
    monkeypatch.setenv("OZGPU_PIPE_FIRST", first)
    got = oz.multiply(a, b, cfg, plan).c
    assert bits_equal(got, want), mismatch_report(got, want)


def test_device_path_graph_replay_is_exact(oz, ref, monkeypatch):
    """ozgpu_dgemm_device replays a captured CUDA graph for repeated calls with
    the same shape, plan, pointers and stream: every replay equals the eager
    result and the reference bitwise, replays read the current contents of
    the inputs, and switching a kernel knob (part of the graph key) is
    honoured."""
    import torch
    rng = np.random.default_rng(11)
    m, k, n = 640, 768, 512
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, 7, 6)
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(device=dev)
    a1, b1 = uniform(m, k, rng), uniform(k, n, rng)
    a2 = uniform(m, k, rng)
    A = torch.from_numpy(a1).to(dev)
    B = torch.from_numpy(b1).to(dev)
    C = torch.empty(m, n, dtype=torch.float64, device=dev)
    want1 = ref_full(ref, a1, b1, 7, 6)
    want2 = ref_full(ref, a2, b1, 7, 6)

    def run():
        oz.multiply_device(m, n, k, A.data_ptr(), k, B.data_ptr(), n, C.data_ptr(), n, cfg, plan,
                           stream=stream.cuda_stream)
        stream.synchronize()
        return C.cpu().numpy()

    monkeypatch.setenv("OZGPU_GRAPH", "1")
    launches = []
    for i in range(4):  # eager, capture, replay, replay
        before = oz.kernel_launches()
        got = run()
        launches.append(oz.kernel_launches() - before)
        assert bits_equal(got, want1), (i, mismatch_report(got, want1))
    assert min(launches) >= 3 and len(set(launches)) == 1, launches
    A.copy_(torch.from_numpy(a2))  # replay must read the new A
    got = run()
    assert bits_equal(got, want2), mismatch_report(got, want2)
    monkeypatch.setenv("OZGPU_CTA_PAIR", "0")  # a different kernel: new graph key
    for _ in range(3):
        got = run()
        assert bits_equal(got, want2), mismatch_report(got, want2)


@pytest.mark.parametrize("m,n,k,slices", [(2304, 2050, 700, (9, 8)), (1800, 2600, 512, (7, 7)),
                                          (3000, 1100, 900, (12, 11)), (8192, 1024, 256, (5, 5))])
def test_split_k_tail_is_exact(oz, ref, m, n, k, slices, monkeypatch):
    """The pair GEMM's split-k tail (the last partial wave's units cut into
    k-ranges whose int32 partial sums are added into pre-zeroed planes)
    returns exactly the un-split result, and the bottom-right blocks (where
    the tail tiles sit) match the reference."""
    rng = np.random.default_rng(m + n + k)
    a = uniform(m, k, rng)
    b = random_matrix(k, n, rng, -5, 5, 0.02)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, *slices)
    monkeypatch.setenv("OZGPU_TAIL_SPLIT", "0")
    want = oz.multiply(a, b, cfg, plan).c
    monkeypatch.setenv("OZGPU_TAIL_SPLIT", "1")
    got = oz.multiply(a, b, cfg, plan).c
    assert bits_equal(got, want), mismatch_report(got, want)
    blocks = [(m - 8, m, n - 8, n), (m - 300, m - 292, n - 270, n - 262), (0, 8, 0, 8)]
    exact, _ = ref.ref_multiply_blocks(a, b, slices[0], slices[1], blocks, 3)
    for r0, r1, c0, c1 in blocks:
        assert bits_equal(got[r0:r1, c0:c1], exact[r0:r1, c0:c1])


@pytest.mark.parametrize("case", ["staged", "below_threshold", "staged_pipeline"])
def test_pageable_staging_is_exact(oz, ref, case, monkeypatch):
    """Pageable host buffers at or above OZGPU_STAGE_MIN bytes are copied by
    host threads into the context's pinned buffers before the GPU pipeline
    (ozgpu_dgemm); smaller products go unstaged.  Either way the result is
    bitwise the unstaged one and matches the reference on sampled blocks --
    incl. a product large enough for the blocked H2D / compute / D2H
    pipeline (the default production route for pageable inputs)."""
    rng = np.random.default_rng(77)
    m, k, n = (2304, 1536, 2048) if case == "staged_pipeline" else (1100, 900, 1300)
    a = uniform(m, k, rng)
    b = random_matrix(k, n, rng, -9, 9, 0.02)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, 8, 7)
    monkeypatch.setenv("OZGPU_STAGE", "0")
    want = oz.multiply(a, b, cfg, plan).c
    monkeypatch.setenv("OZGPU_STAGE", "1")
    total = 8 * (m * k + k * n + m * n)
    monkeypatch.setenv("OZGPU_STAGE_MIN", str(total + 1) if case == "below_threshold" else "0")
    got = oz.multiply(a, b, cfg, plan).c
    assert bits_equal(got, want), mismatch_report(got, want)
    blocks = [(0, 8, 0, 8), (m - 8, m, n - 8, n)]
    exact, _ = ref.ref_multiply_blocks(a, b, 8, 7, blocks, 2)
    for r0, r1, c0, c1 in blocks:
        assert bits_equal(got[r0:r1, c0:c1], exact[r0:r1, c0:c1])


def test_underflow_regime(oz, ref, po):
    """Scaled products below 2^-1022 (scheme.cpp:205-215): the reference
    rounds every pair term onto the subnormal grid inside ldexp before its
    (otherwise exact) level sums, so it can miss RN(exact) by a few units of
    2^-1074; the GPU computes the exact scheduled sum and rounds once.
    Shown here: in the error-free regime (slices hold A and B exactly) the
    GPU equals the exact product RN(AB) bit for bit -- as the C restatement of
    the levelled-exact contract does -- and the reference stays within
    (terms + 1) / 2 units of 2^-1074 of it; with truncating slices both stay
    inside the a13 bound plus that underflow allowance."""
    rng = np.random.default_rng(1)
    cfg = oz.MmaConfig.int8_int32()
    tiny = 2.0 ** -1074
    m, k, n = 24, 40, 20
    a = np.ldexp(rng.integers(-2**13, 2**13, size=(m, k)).astype(np.float64), -540)
    b = np.ldexp(rng.integers(-2**13, 2**13, size=(k, n)).astype(np.float64), -540)
    a[3] *= 2.0 ** 500  # a row of normal-range products next to subnormal ones
    exact = ref.ref_exact_gemm(a, b)
    assert (np.abs(exact[:3]) < 2.0 ** -1022).all()
    for sa, sb, sched in [(4, 4, 0), (4, 4, 1), (3, 3, 0)]:
        plan = oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind(sched))
        got = oz.multiply(a, b, cfg, plan).c
        assert bits_equal(got, exact), mismatch_report(got, exact)
        assert bits_equal(got, po.port_multiply_exact(a, b, sa, sb, sched))
        want, diag = ref.ref_multiply(a, b, sa, sb, sched)
        terms = diag[0]
        assert (np.abs(want - exact) <= (terms + 1) * tiny / 2).all()
    # truncating slices (uniform magnitudes, s = 2): both inside the bound
    a2 = a * np.exp(rng.uniform(-3, 3, size=a.shape))
    b2 = b * np.exp(rng.uniform(-3, 3, size=b.shape))
    for sa, sb in [(2, 2), (3, 2)]:
        plan = oz.make_plan(cfg, k, sa, sb)
        got = oz.multiply(a2, b2, cfg, plan).c
        want, diag = ref.ref_multiply(a2, b2, sa, sb)
        rep = oz.error_bound(a2, b2, plan)
        ex2 = ref.ref_exact_gemm(a2, b2)
        allow = rep.bound + (diag[0] + 1) * tiny / 2
        assert (np.abs(got - ex2) <= allow).all()
        assert (np.abs(want - ex2) <= allow).all()
        assert bits_equal(got, po.port_multiply_exact(a2, b2, sa, sb))

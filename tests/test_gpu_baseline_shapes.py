"""Parity at the BASELINE.json shapes on the production kernels.

* The int8 slicer hook (ozgpu_split_i8) runs exactly the launches multiply()
  makes for its operands (rowmax + streaming row slicer, column max +
  transposing column slicer) at full size; sampled rows / columns must equal
  the reference's split() bit for bit (slicing.cpp:67-132).
* The pair-planes hook (ozgpu_pair_planes) runs the production tcgen05
  CTA-pair GEMM (chunk bins, wave lockstep, split-k tail) at full size; every
  chunk plane in sampled windows must equal the exact sum of the reference's
  integer_gemm products of its slice pairs (mma_sim.cpp:76-125), computed
  here from the reference's own slices.
* multiply() at full size: sampled C blocks (incl. the ragged / split-k tail
  corner) equal the reference multiply() on the same blocks bit for bit --
  blocking is exact because the scales are per row of A / column of B
  (SURVEY.md fact 5).

configs[2] 4096^3 gen_kappa_d(2^60, seed 7, rotate) at the estimator's
(16,17) and the gamma_psi choice (17,17); configs[3] 65536 x 2048^2 at
(12,11); m = n = 2048 with k = 16384 (13,12) (int32 capacity 8 pairs per
chunk: multi-chunk diagonals) and k = 32768 (capacity 4, consecutive-cut bins)
under the plane-budget row blocking.
"""
import numpy as np
import pytest

from helpers import bits_equal, mismatch_report

pytestmark = pytest.mark.gpu

T = 7


def _check_slices_rows(oz, ref, a, count, rows):
    out, scales = oz.split_i8(a, T, count, oz.BlockOrientation.ROWS)
    k = a.shape[1]
    wsc, wsl = ref.ref_split(a[rows], 0, T, count)
    assert np.array_equal(scales[rows], wsc)
    got = out[:, rows, :k].astype(np.int64)
    assert np.array_equal(got, wsl), int(np.sum(got != wsl))
    assert not out[:, rows, k:].any()  # zero-filled K tail


def _check_slices_cols(oz, ref, b, count, cols):
    out, scales = oz.split_i8(b, T, count, oz.BlockOrientation.COLUMNS)
    k = b.shape[0]
    wsc, wsl = ref.ref_split(b[:, cols], 1, T, count)
    assert np.array_equal(scales[cols], wsc)
    got = out[:, cols, :k].astype(np.int64)  # K-major: [slice][column][k]
    assert np.array_equal(got, np.transpose(wsl, (0, 2, 1))), int(np.sum(got != wsl.transpose(0, 2, 1)))
    assert not out[:, cols, k:].any()


def _check_planes(oz, ref, a, b, plan, windows):
    """Each chunk plane == sum over its pairs of E_lh = A_l B_h (exact
    integers: |partial sums| < 2^31, so a float64 product is exact)."""
    cfg = oz.MmaConfig.int8_int32()
    sa, sb = plan.slices_a, plan.slices_b
    for win in windows:
        r0, r1, c0, c1 = win
        planes, chunks = oz.pair_planes(a, b, cfg, plan, win)
        _, sla = ref.ref_split(a[r0:r1], 0, plan.width, sa)
        _, slb = ref.ref_split(b[:, c0:c1], 1, plan.width, sb)
        fa, fb = sla.astype(np.float64), slb.astype(np.float64)
        pairs = 0
        for c, (d, l0, npairs) in enumerate(chunks):
            want = np.zeros((r1 - r0, c1 - c0))
            for p in range(npairs):
                l, h = l0 + p, d + 2 - (l0 + p)
                want += fa[l - 1] @ fb[h - 1]
            pairs += npairs
            assert np.array_equal(planes[c].astype(np.int64), want.astype(np.int64)), \
                (win, c, d, l0, npairs, int(np.sum(planes[c] != want)))
        if plan.schedule == oz.ScheduleKind.REDUCED:
            assert pairs == oz.chi(sa, sb)


def _check_blocks(oz, ref, a, b, c, plan, blocks, threads=8):
    want, _ = ref.ref_multiply_blocks(a, b, plan.slices_a, plan.slices_b, blocks, threads)
    for r0, r1, c0, c1 in blocks:
        assert bits_equal(c[r0:r1, c0:c1], want[r0:r1, c0:c1]), \
            ((r0, c0), mismatch_report(c[r0:r1, c0:c1], want[r0:r1, c0:c1]))


@pytest.fixture(scope="module")
def kappa_d(oz):
    return oz.gen_kappa_d(4096, 2.0 ** 60, 7, True)


def test_configs2_kappa_d_estimator_choice(oz, ref, kappa_d):
    """configs[2]: the GPU kappa scan + host estimator choose what the
    reference chooses: (16,17) at 1e-15, (17,17) at the default gamma_psi."""
    a, b = kappa_d
    prof = oz.scaling_profile(a, b)
    ka, kb, za, zb = ref.ref_scaling_profile(a, b)
    assert (prof.kappa_a, prof.kappa_b) == (ka, kb)
    acc = 2 * T + 12
    sel = oz.select_slices(prof.kappa_a, prof.kappa_b, T, 2.0 ** -53, 24,
                           oz.SelectOptions(target=1e-15, acc_bits_used=acc))
    assert (sel.slices_a, sel.slices_b) == (16, 17)
    wsel = ref.ref_select_slices(ka, kb, T, 2.0 ** -53, 24, target=1e-15, acc_bits_used=acc)
    assert (wsel["slices_a"], wsel["slices_b"]) == (16, 17)
    sel2 = oz.select_slices(prof.kappa_a, prof.kappa_b, T, 2.0 ** -53, 24,
                            oz.SelectOptions(acc_bits_used=acc))
    wsel2 = ref.ref_select_slices(ka, kb, T, 2.0 ** -53, 24, acc_bits_used=acc)
    assert (sel2.slices_a, sel2.slices_b) == (wsel2["slices_a"], wsel2["slices_b"]) == (17, 17)


@pytest.mark.parametrize("queue", ["0", "1"])
def test_configs2_kappa_d_slices(oz, ref, kappa_d, queue, monkeypatch):
    monkeypatch.setenv("OZGPU_SLICE_QUEUE", queue)  # two-kernel (default) / one-launch queue slicer
    a, b = kappa_d
    sample = [0, 1, 777, 2048, 4000, 4095]
    _check_slices_rows(oz, ref, a, 16, sample)
    _check_slices_cols(oz, ref, b, 17, sample)


@pytest.mark.parametrize("slices", [(16, 17), (17, 17)])
def test_configs2_kappa_d_planes_and_c(oz, ref, kappa_d, slices):
    a, b = kappa_d
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, 4096, *slices)
    _check_planes(oz, ref, a, b, plan, [(0, 24, 0, 24), (4072, 4096, 4072, 4096),
                                        (1900, 1924, 3000, 3024)])
    c = oz.multiply(a, b, cfg, plan).c
    _check_blocks(oz, ref, a, b, c, plan, [(0, 16, 0, 16), (4080, 4096, 4080, 4096),
                                           (4080, 4096, 0, 16), (2040, 2056, 2040, 2056)])


def test_configs3_tall_skinny(oz, ref):
    """configs[3]: 65536 x 2048 x 2048 at the estimator's (12, 11)."""
    m, n, k = 65536, 2048, 2048
    a = oz.random_uniform(m, k, 1, -0.5, 0.5)
    b = oz.random_uniform(k, n, 2, -0.5, 0.5)
    cfg = oz.MmaConfig.int8_int32()
    prof = oz.scaling_profile(a, b)
    sel = oz.select_slices(prof.kappa_a, prof.kappa_b, T, 2.0 ** -53, 24,
                           oz.SelectOptions(target=1e-15, acc_bits_used=2 * T + 11))
    assert (sel.slices_a, sel.slices_b) == (12, 11)
    _check_slices_rows(oz, ref, a, 12, [0, 5, 32767, 65535])
    _check_slices_cols(oz, ref, b, 11, [0, 1000, 2047])
    plan = oz.make_plan(cfg, k, 12, 11)
    _check_planes(oz, ref, a, b, plan, [(65512, 65536, 2024, 2048), (30000, 30024, 100, 124)])
    c = oz.multiply(a, b, cfg, plan).c
    _check_blocks(oz, ref, a, b, c, plan, [(0, 16, 0, 16), (65520, 65536, 2032, 2048),
                                           (40000, 40016, 1024, 1040), (65520, 65536, 0, 16)])


def test_multi_chunk_diagonals_k16384(oz, ref):
    """m = n = 2048, k = 16384 at the north star's (13, 12): int32 capacity 8
    pairs per chunk, so the 12-pair diagonals run as two chunks each on the
    CTA-pair kernel with bins, lockstep and the split-k tail."""
    m, n, k = 2048, 2048, 16384
    a = oz.random_uniform(m, k, 1, -0.5, 0.5)
    b = oz.random_uniform(k, n, 2, -0.5, 0.5)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, 13, 12)
    planes, chunks = oz.pair_planes(a, b, cfg, plan, (0, 1, 0, 1))
    assert max(c[2] for c in chunks) == 8 and len(chunks) > 13
    _check_planes(oz, ref, a, b, plan, [(2032, 2048, 2032, 2048), (0, 16, 1024, 1040)])
    c = oz.multiply(a, b, cfg, plan).c
    _check_blocks(oz, ref, a, b, c, plan, [(0, 16, 0, 16), (2032, 2048, 2032, 2048),
                                           (1000, 1016, 1500, 1516)])


def test_k32768_plane_budget_row_blocks(oz, ref, monkeypatch):
    """k = 32768 (capacity 4 pairs per chunk: 27 chunks at (13,12), bins cut
    consecutively) with the chunk-plane budget forcing row blocks of C."""
    m, n, k = 2048, 2048, 32768
    a = oz.random_uniform(m, k, 1, -0.5, 0.5)
    b = oz.random_uniform(k, n, 2, -0.5, 0.5)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, 13, 12)
    _, chunks = oz.pair_planes(a, b, cfg, plan, (0, 1, 0, 1))
    assert len(chunks) == 27 and max(c[2] for c in chunks) == 4
    # one whole-matrix run_multiply (no host pipeline) whose 27 planes (0.42
    # GiB) exceed the budget -> GEMM + combine over 512-row blocks of C
    monkeypatch.setenv("OZGPU_PIPE", "0")
    monkeypatch.setenv("OZGPU_PLANE_BUDGET_GB", "0.15")
    c = oz.multiply(a, b, cfg, plan).c
    monkeypatch.delenv("OZGPU_PLANE_BUDGET_GB")
    monkeypatch.delenv("OZGPU_PIPE")
    c_unblocked = oz.multiply(a, b, cfg, plan).c  # default route: the blocked host pipeline
    assert bits_equal(c, c_unblocked), mismatch_report(c, c_unblocked)
    _check_blocks(oz, ref, a, b, c, plan, [(0, 16, 0, 16), (2032, 2048, 2032, 2048),
                                           (700, 716, 300, 316)], threads=3)


def _edge_rows(rng, k):
    """Rows that walk the production slicer's exponent edges: entries from
    the block max down past 2^-64 and 2^-128 of it (window-1 shift directions,
    a0 = 64 exactly), subnormals inside a normal row, block maxima around
    2^-1000 (the t = 7 fast emit needs q >= -1000; below it the generic one
    runs), all-subnormal and huge rows, zeros, and random-exponent rows."""
    rows = []
    e = np.arange(k) % 140
    r = np.ldexp(1.0 + rng.random(k), -e)
    r[0] = 1.5
    rows.append(r)
    rows.append(-r[::-1] * np.where(rng.random(k) < 0.5, 1.0, -1.0))
    r = np.ldexp(0.5 + rng.random(k) / 2, rng.integers(-20, 1, k))
    r[::7] = np.ldexp(1.0, -1060) * (1 + np.arange(len(r[::7])))  # subnormals in a normal row
    rows.append(r)
    r = np.ldexp(1.0, 64 - np.arange(k) % 66)  # exact powers: a0 = 0 .. 65 around 64
    rows.append(r * np.where(np.arange(k) % 3 == 0, -1.0, 1.0))
    for top in (-1001, -1002, -1003):  # q = -1000 (fast emit), -1001, -1002 (generic)
        r = np.ldexp(1.0 + rng.random(k), top - rng.integers(0, 60, k))
        r[1] = np.ldexp(1.5, top)
        rows.append(r * np.where(rng.random(k) < 0.5, 1.0, -1.0))
    rows.append(np.ldexp(1.0 + np.arange(k), -1074 + 10) * np.where(np.arange(k) % 2, 1.0, -1.0))
    r = np.ldexp(1.0 + rng.random(k), 1020 - rng.integers(0, 200, k))
    rows.append(r)
    rows.append(np.zeros(k))
    for _ in range(6):
        rows.append(np.ldexp(rng.random(k) - 0.5, rng.integers(-80, 80, k)))
    x = np.array(rows)
    x[x == 0] = 0.0  # no -0 (rejected inputs)
    return x


@pytest.mark.parametrize("count", [1, 4, 9, 10, 12, 13, 14, 17])
@pytest.mark.parametrize("k", [200, 201])
def test_production_slicer_exponent_edges(oz, ref, count, k):
    """The production int8 slicers (rows and columns; k = 200 takes the
    vectorised kernels with a compile-time slice count, k = 201 the scalar
    ones) bit-exact against the reference's split() on rows built to hit
    every branch of the windowed extraction."""
    rng = np.random.default_rng(count * 1000 + k)
    x = _edge_rows(rng, k)
    idx = np.arange(x.shape[0])
    _check_slices_rows(oz, ref, x, count, idx)
    _check_slices_cols(oz, ref, np.ascontiguousarray(x.T), count, idx)

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

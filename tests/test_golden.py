"""Golden fixtures generated from the unmodified reference
(tests/golden/make_golden.py): the C restatement (CPU) and the CUDA path
(GPU) reproduce them bit-for-bit."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import ROOT
from helpers import bits_equal, mismatch_report

GOLD = os.path.join(ROOT, "tests", "golden")


def _cases():
    z = np.load(os.path.join(GOLD, "small.npz"))
    return [{key: z[f"{i}_{key}"] for key in ("a", "b", "plan", "c", "diag")}
            for i in range(int(z["count"]))]


def test_oracle_reproduces_small_golden(po):
    n = 0
    for cs in _cases():
        sa, sb, sched, strat, mode = (int(v) for v in cs["plan"])
        if strat != 2:
            continue  # the restatement covers the default levelled-exact strategy
        got = po.port_multiply_exact(cs["a"], cs["b"], sa, sb, schedule=sched, mode=mode)
        assert bits_equal(got, cs["c"])
        n += 1
    assert n >= 20


def test_config1_inputs_match_golden(po):
    meta = json.load(open(os.path.join(GOLD, "config1.json")))
    a = po.port_random_uniform(1024, 1024, 1, -0.5, 0.5)
    b = po.port_random_uniform(1024, 1024, 2, -0.5, 0.5)
    assert hashlib.sha256(a.tobytes()).hexdigest() == meta["sha256_a"]
    assert hashlib.sha256(b.tobytes()).hexdigest() == meta["sha256_b"]


@pytest.mark.gpu
def test_gpu_reproduces_small_golden(oz):
    cfg = oz.MmaConfig.int8_int32()
    for cs in _cases():
        sa, sb, sched, strat, mode = (int(v) for v in cs["plan"])
        k = cs["a"].shape[1]
        plan = oz.make_plan(cfg, k, sa, sb, oz.ScheduleKind(sched), oz.Accumulation(strat),
                            oz.SliceMode(mode))
        r = oz.multiply(cs["a"], cs["b"], cfg, plan)
        assert bits_equal(r.c, cs["c"]), (cs["plan"], mismatch_report(r.c, cs["c"]))
        d = r.diagnostics
        assert [d.products, d.integer_adds, d.float_adds, d.flushes, d.realized_psi,
                d.planned_psi, d.width, d.acc_bits_used] == cs["diag"].tolist()


@pytest.mark.gpu
def test_gpu_config1_bit_exact(oz):
    """configs[0] in full: 1024^3, s=(4,4) -- sha256 of C equals the reference's."""
    meta = json.load(open(os.path.join(GOLD, "config1.json")))
    cfg = oz.MmaConfig.int8_int32()
    a = oz.random_uniform(1024, 1024, 1, -0.5, 0.5)
    b = oz.random_uniform(1024, 1024, 2, -0.5, 0.5)
    c = oz.multiply(a, b, cfg, oz.make_plan(cfg, 1024, 4, 4)).c
    for s in meta["samples"]:
        r0, c0 = s["row0"], s["col0"]
        assert bits_equal(c[r0:r0 + 32, c0:c0 + 32], np.array(s["c"]))
    assert hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest() == meta["sha256_c_f64_le"]

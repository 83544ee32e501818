"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libozref.so, compiled from /root/reference/proj).

    python tests/golden/make_golden.py

* small.npz       -- small multiply cases (inputs, plan, C, Diagnostics) across
                     schedules, modes, strategies and scalings
* config1.json    -- configs[0] (m=n=k=1024, uniform(-0.5,0.5) seeds 1/2,
                     s=(4,4), reduced, levelled-exact): sha256 of the reference C
                     bytes plus 4 sampled 32x32 blocks
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402


def rmat(rows, cols, rng, lo, hi, zf=0.0):
    frac = rng.integers(0, 2**53, size=(rows, cols), dtype=np.int64).astype(np.float64) * 2.0**-53
    e = rng.integers(lo, hi + 1, size=(rows, cols))
    x = np.ldexp(1.0 + frac, e) * np.where(rng.integers(0, 2, size=(rows, cols)) == 1, 1.0, -1.0)
    if zf:
        x[rng.random((rows, cols)) < zf] = 0.0
    return x


def small_cases():
    rng = np.random.default_rng(2025)
    cases = []
    shapes = [(1, 1, 1), (4, 7, 5), (16, 33, 9), (31, 64, 17)]
    plans = [(4, 4, 1, 2, 0), (8, 8, 1, 2, 0), (3, 7, 0, 2, 0), (6, 6, 1, 2, 1), (5, 5, 1, 0, 0),
             (5, 5, 0, 1, 1), (13, 12, 1, 2, 0)]
    for (m, k, n) in shapes:
        for sa, sb, sched, strat, mode in plans:
            a = rmat(m, k, rng, -20, 20, 0.05)
            b = rmat(k, n, rng, -20, 20, 0.05)
            c, diag = po.ref_multiply(a, b, sa, sb, sched, strat, mode)
            cases.append(dict(a=a, b=b, plan=np.array([sa, sb, sched, strat, mode]), c=c, diag=diag))
    a, b = po.ref_gen_kappa_d(24, 2.0**60, 7, True)
    for sa, sb in [(8, 8), (16, 17)]:
        c, diag = po.ref_multiply(a, b, sa, sb)
        cases.append(dict(a=a, b=b, plan=np.array([sa, sb, 1, 2, 0]), c=c, diag=diag))
    return cases


def main():
    cases = small_cases()
    flat = {}
    for i, cs in enumerate(cases):
        for key, v in cs.items():
            flat[f"{i}_{key}"] = v
    flat["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "small.npz"), **flat)

    n = 1024
    a = po.ref_random_uniform(n, n, 1, -0.5, 0.5)
    b = po.ref_random_uniform(n, n, 2, -0.5, 0.5)
    bs = 128
    blocks = [(i, i + bs, j, j + bs) for i in range(0, n, bs) for j in range(0, n, bs)]
    c, secs = po.ref_multiply_blocks(a, b, 4, 4, blocks, os.cpu_count() or 1)
    assert not np.isnan(c).any()
    samples = []
    for (r, q) in [(0, 0), (517, 93), (960, 992), (300, 700)]:
        samples.append({"row0": r, "col0": q, "c": c[r:r + 32, q:q + 32].tolist()})
    meta = {"workload": "configs[0]: m=n=k=1024, uniform(-0.5,0.5) seeds 1,2, s=(4,4), reduced, "
                        "levelled-exact, truncate",
            "sha256_c_f64_le": hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest(),
            "sha256_a": hashlib.sha256(a.tobytes()).hexdigest(),
            "sha256_b": hashlib.sha256(b.tobytes()).hexdigest(),
            "reference_seconds": secs, "blocks": f"{len(blocks)} blocks of {bs}x{bs}",
            "samples": samples}
    with open(os.path.join(HERE, "config1.json"), "w") as f:
        json.dump(meta, f)
    print(f"wrote {len(cases)} small cases; config1 reference time {secs:.1f} s")


if __name__ == "__main__":
    main()

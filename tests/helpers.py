"""Shared input builders (mirroring the reference tests' fixed-seed builders,
e.g. proj/tests/scheme_test.cpp:44-54)."""
import numpy as np


def random_matrix(rows, cols, rng, exp_lo=-4, exp_hi=4, zero_frac=0.0):
    """(1 + frac) * 2^e * sign with e uniform in [exp_lo, exp_hi]."""
    frac = rng.integers(0, 2**53, size=(rows, cols), dtype=np.int64).astype(np.float64) * 2.0**-53
    e = rng.integers(exp_lo, exp_hi + 1, size=(rows, cols))
    sign = np.where(rng.integers(0, 2, size=(rows, cols)) == 1, 1.0, -1.0)
    out = np.ldexp(1.0 + frac, e) * sign
    if zero_frac:
        out[rng.random((rows, cols)) < zero_frac] = 0.0
    return out


def uniform(rows, cols, rng, lo=-0.5, hi=0.5):
    return lo + rng.random((rows, cols)) * (hi - lo)


def bits_equal(x, y) -> bool:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))


def mismatch_report(x, y, limit=5) -> str:
    x = np.asarray(x)
    y = np.asarray(y)
    bad = np.argwhere(x.view(np.uint64) != y.view(np.uint64))
    rows = [f"{tuple(i)}: got {x[tuple(i)]!r} want {y[tuple(i)]!r}" for i in bad[:limit]]
    return f"{len(bad)} mismatches; " + "; ".join(rows)


def ref_full(ref, a, b, sa, sb, schedule=1, strategy=2, mode=0):
    """The reference multiply() of the whole product, run as row blocks of C on
    every host core (bit-identical to one call: each element's computation is
    independent of the others and the scales are per row / column)."""
    import os
    m, n = a.shape[0], b.shape[1]
    threads = os.cpu_count() or 4
    parts = max(1, min(m, 2 * threads))
    blocks = [(m * i // parts, m * (i + 1) // parts, 0, n) for i in range(parts)
              if m * i // parts < m * (i + 1) // parts]
    c, _ = ref.ref_multiply_blocks(a, b, sa, sb, blocks, threads, schedule, strategy, mode)
    return c

"""Host-buffer multiply from pinned vs pageable (plain numpy) memory, and the
cost of cudaHostRegister on the pageable buffers (development tool).

Usage: python tools/pageable_probe.py [--n 8192] [--s 12 12] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_11277_b200 as oz  # noqa: E402


def timed(fn, steps):
    fn()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    return (time.perf_counter() - t0) / steps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--s", type=int, nargs=2, default=[12, 12])
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    n = a.n
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, n, *a.s)
    A = oz.random_uniform(n, n, 1, -0.5, 0.5)
    B = oz.random_uniform(n, n, 2, -0.5, 0.5)
    C = np.empty((n, n))
    Ap = torch.from_numpy(A).pin_memory().numpy()
    Bp = torch.from_numpy(B).pin_memory().numpy()
    Cp = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
    out = {"n": n}
    out["pinned_ms"] = timed(lambda: oz.multiply(Ap, Bp, cfg, plan, out=Cp), a.steps)
    out["pageable_ms"] = timed(lambda: oz.multiply(A, B, cfg, plan, out=C), a.steps)
    assert np.array_equal(C.view(np.uint64), Cp.view(np.uint64))
    rt = torch.cuda.cudart()
    t0 = time.perf_counter()
    for x in (A, B, C):
        rt.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    out["register_ms"] = (time.perf_counter() - t0) * 1e3
    out["registered_ms"] = timed(lambda: oz.multiply(A, B, cfg, plan, out=C), a.steps)
    t0 = time.perf_counter()
    for x in (A, B, C):
        rt.cudaHostUnregister(x.ctypes.data)
    out["unregister_ms"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

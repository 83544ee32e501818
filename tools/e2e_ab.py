"""A/B of the host-pointer path (ozgpu_dgemm: H2D + compute + D2H) for env
variants, interleaved rounds (development tool).

Usage: python tools/e2e_ab.py [--n 8192] [--s 12 12] [--steps 4] [--rounds 3] VAR=V,VAR=V ...
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_11277_b200 as oz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--s", type=int, nargs=2, default=[12, 12])
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--pageable", action="store_true", help="plain numpy buffers (staged path)")
    ap.add_argument("variants", nargs="*", default=[""])
    a = ap.parse_args()
    n, k, m = a.n, a.k or a.n, a.m or a.n
    if a.pageable:
        A = oz.random_uniform(m, k, 1, -0.5, 0.5)
        B = oz.random_uniform(k, n, 2, -0.5, 0.5)
        C = np.empty((m, n), dtype=np.float64)
    else:
        A = torch.from_numpy(oz.random_uniform(m, k, 1, -0.5, 0.5)).pin_memory().numpy()
        B = torch.from_numpy(oz.random_uniform(k, n, 2, -0.5, 0.5)).pin_memory().numpy()
        C = torch.empty((m, n), dtype=torch.float64).pin_memory().numpy()
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, *a.s)
    ref = None
    res = {v: [] for v in a.variants}
    same = {v: True for v in a.variants}
    for _ in range(a.rounds):
        for var in a.variants:
            env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
            saved = {key: os.environ.get(key) for key in env}
            os.environ.update(env)
            oz.multiply(A, B, cfg, plan, out=C)
            if ref is None:
                ref = C.copy()
            same[var] &= bool(np.array_equal(C.view(np.uint64), ref.view(np.uint64)))
            t0 = time.perf_counter()
            for _ in range(a.steps):
                oz.multiply(A, B, cfg, plan, out=C)
            res[var].append((time.perf_counter() - t0) / a.steps * 1e3)
            for key, v in saved.items():
                if v is None:
                    os.environ.pop(key, None)
                else:
                    os.environ[key] = v
    for var in a.variants:
        ms = statistics.median(res[var])
        print(json.dumps({"variant": var or "default", "e2e_ms": ms,
                          "tflops": 2.0 * m * n * k / (ms * 1e-3) / 1e12,
                          "rounds": [round(x, 2) for x in res[var]], "same_as_first": same[var]}),
              flush=True)


if __name__ == "__main__":
    main()

"""A/B of the slicing stage (device-resident multiply, eager with stage
timing) for env variants, interleaved rounds (development tool).

Usage: python tools/slice_ab.py [--n 8192] [--s 12 12] [--steps 4] [--rounds 3] VAR=V,VAR=V ...
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_11277_b200 as oz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--m", type=int, default=0, help="rows of A (default n)")
    ap.add_argument("--k", type=int, default=0, help="inner dimension (default n)")
    ap.add_argument("--s", type=int, nargs=2, default=[12, 12])
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("variants", nargs="*", default=[""])
    a = ap.parse_args()
    n = a.n
    m = a.m or n
    k = a.k or n
    A = torch.from_numpy(oz.random_uniform(m, k, 1, -0.5, 0.5)).cuda()
    B = torch.from_numpy(oz.random_uniform(k, n, 2, -0.5, 0.5)).cuda()
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, *a.s)
    oz.set_stage_timing(True)
    ref = None
    res = {v: [] for v in a.variants}
    same = {v: True for v in a.variants}

    def call():
        oz.multiply_device(m, n, k, A.data_ptr(), k, B.data_ptr(), n, C.data_ptr(), n, cfg, plan,
                           stream=torch.cuda.current_stream().cuda_stream)

    for _ in range(a.rounds):
        for var in a.variants:
            env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
            saved = {key: os.environ.get(key) for key in env}
            os.environ.update(env)
            call()
            torch.cuda.synchronize()
            if ref is None:
                ref = C.clone()
            same[var] &= bool(torch.equal(C.view(torch.int64), ref.view(torch.int64)))
            oz.stage_times(reset=True)
            for _ in range(a.steps):
                call()
            torch.cuda.synchronize()
            sl, gm, cb, calls = oz.stage_times(reset=True)
            res[var].append((sl / calls, gm / calls, cb / calls))
            for key, v in saved.items():
                if v is None:
                    os.environ.pop(key, None)
                else:
                    os.environ[key] = v
    for var in a.variants:
        print(json.dumps({"variant": var or "default",
                          "slicing_ms": statistics.median(r[0] for r in res[var]),
                          "gemm_ms": statistics.median(r[1] for r in res[var]),
                          "combine_ms": statistics.median(r[2] for r in res[var]),
                          "slicing_rounds": [round(r[0], 3) for r in res[var]],
                          "same_as_first": same[var]}), flush=True)


if __name__ == "__main__":
    main()

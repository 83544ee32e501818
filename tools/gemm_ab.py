"""A/B timing of GEMM-path variants on one GPU (development tool).

Usage: python tools/gemm_ab.py [--n 8192] [--s 12] [--steps 5] VAR=VAL,VAR=VAL ...
Each argument is one variant: a comma-separated list of OZGPU_* env settings
(read by the library per call).  Prints per-stage device times per variant.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_11277_b200 as oz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--s", type=int, nargs=2, default=[12, 12])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("variants", nargs="*", default=[""])
    a = ap.parse_args()
    n, k = a.n, a.k or a.n
    dev = torch.device("cuda:0")
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    A = torch.from_numpy(oz.random_uniform(n, k, 1, -0.5, 0.5)).to(dev)
    B = torch.from_numpy(oz.random_uniform(k, n, 2, -0.5, 0.5)).to(dev)
    C = torch.empty(n, n, dtype=torch.float64, device=dev)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, *a.s)
    chi = oz.chi(*a.s)
    ref = None
    out = []
    for var in a.variants:
        env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
        saved = {key: os.environ.get(key) for key in env}
        os.environ.update(env)
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(2):
            oz.multiply_device(n, n, k, A.data_ptr(), k, B.data_ptr(), n, C.data_ptr(), n, cfg,
                               plan, stream=st)
        torch.cuda.synchronize()
        if ref is None:
            ref = C.clone()
        same = bool(torch.equal(C.view(torch.int64), ref.view(torch.int64)))
        oz.stage_times(reset=True)
        oz.set_stage_timing(True)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            oz.multiply_device(n, n, k, A.data_ptr(), k, B.data_ptr(), n, C.data_ptr(), n, cfg,
                               plan, stream=st)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / a.steps
        oz.set_stage_timing(False)
        s_ms, g_ms, c_ms, calls = oz.stage_times(reset=True)
        calls = max(calls, 1)
        rec = {"variant": var or "default", "slicing_ms": s_ms / calls, "gemm_ms": g_ms / calls,
               "combine_ms": c_ms / calls, "wall_ms": wall * 1e3,
               "int8_tops": 2.0 * chi * n * n * k / (g_ms / calls * 1e-3) / 1e12,
               "fp64_equiv_tflops": 2.0 * n * n * k / wall / 1e12, "same_as_first": same}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        for key, v in saved.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


if __name__ == "__main__":
    main()

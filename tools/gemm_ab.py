"""A/B timing of GEMM-path variants on one GPU (development tool).

Usage: python tools/gemm_ab.py [--n 8192] [--s 12 12] [--steps 10] [--rounds 3] VAR=VAL,VAR=VAL ...
Each argument is one variant: a comma-separated list of OZGPU_* env settings
(read by the library per call).  Variants are interleaved round by round
(A B C A B C ...) so the power-capped clock affects them alike; per variant
the median over rounds of the per-stage device times is printed, with the SM
clock and board power sampled through NVML while it ran.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_11277_b200 as oz  # noqa: E402


class Sampler:
    def __init__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        except Exception:
            self.nv = None
        self.samples = []
        self.stop_ev = threading.Event()

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                clk = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                pw = self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((clk, pw))
            except Exception:
                pass
            time.sleep(0.02)

    def start(self):
        self.samples = []
        self.stop_ev.clear()
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if not self.nv:
            return None, None
        self.stop_ev.set()
        self.t.join()
        if not self.samples:
            return None, None
        return (statistics.median(s[0] for s in self.samples),
                statistics.median(s[1] for s in self.samples))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--s", type=int, nargs=2, default=[12, 12])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("variants", nargs="*", default=[""])
    a = ap.parse_args()
    n, k, m = a.n, a.k or a.n, a.m or a.n
    dev = torch.device("cuda:0")
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    A = torch.from_numpy(oz.random_uniform(m, k, 1, -0.5, 0.5)).to(dev)
    B = torch.from_numpy(oz.random_uniform(k, n, 2, -0.5, 0.5)).to(dev)
    C = torch.empty(m, n, dtype=torch.float64, device=dev)
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, *a.s)
    chi = oz.chi(*a.s)
    ref = None
    res = {v: [] for v in a.variants}
    same = {v: True for v in a.variants}
    sampler = Sampler()
    st = torch.cuda.current_stream().cuda_stream

    def run(nsteps):
        for _ in range(nsteps):
            oz.multiply_device(m, n, k, A.data_ptr(), k, B.data_ptr(), n, C.data_ptr(), n, cfg,
                               plan, stream=st)

    for rnd in range(a.rounds):
        for var in a.variants:
            env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
            saved = {key: os.environ.get(key) for key in env}
            os.environ.update(env)
            run(1)
            torch.cuda.synchronize()
            if ref is None:
                ref = C.clone()
            same[var] &= bool(torch.equal(C.view(torch.int64), ref.view(torch.int64)))
            oz.stage_times(reset=True)
            oz.set_stage_timing(True)
            sampler.start()
            t0 = time.perf_counter()
            run(a.steps)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / a.steps
            clk, pw = sampler.stop()
            oz.set_stage_timing(False)
            s_ms, g_ms, c_ms, calls = oz.stage_times(reset=True)
            calls = max(calls, 1)
            res[var].append({"slicing_ms": s_ms / calls, "gemm_ms": g_ms / calls,
                             "combine_ms": c_ms / calls, "wall_ms": wall * 1e3,
                             "sm_mhz": clk, "power_w": pw})
            for key, v in saved.items():
                if v is None:
                    os.environ.pop(key, None)
                else:
                    os.environ[key] = v
    for var in a.variants:
        rows = res[var]
        med = {key: statistics.median(r[key] for r in rows if r[key] is not None)
               if any(r[key] is not None for r in rows) else None for key in rows[0]}
        med["int8_tops"] = 2.0 * chi * m * n * k / (med["gemm_ms"] * 1e-3) / 1e12
        med["fp64_equiv_tflops"] = 2.0 * m * n * k / (med["wall_ms"] * 1e-3) / 1e12
        med["gemm_ms_rounds"] = [round(r["gemm_ms"], 3) for r in rows]
        print(json.dumps({"variant": var or "default", **med, "same_as_first": same[var]}),
              flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Benchmark of the B200-native Ozaki-I FP64 GEMM (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Metric (BASELINE.json): effective FP64-equivalent TFLOP/s = 2mnk / t, with
the int8 tensor-pipe rate of the pair GEMMs (2*chi*mnk / t_gemm) reported
against the int8 dense peak as the roofline.

Workload at N=1: configs[1] -- FP64 GEMM m=n=k=8192, uniform(-0.5, 0.5) inputs
from the reference generator (seeds 1 and 2), slice counts chosen by the
reference's estimator for a 1e-15 target -> (12, 12), chi=78;
the s=3..8 sweep of the same config is reported beside it.

N > 1 (torchrun, one process per GPU, NCCL): weak scaling with 2-D C tiles --
rank (i, j) computes an m x n block of a (p_r m) x (p_c n) product with the
full k; A row-panel i lives on rank (i, 0) and B column-panel j on (0, j) and
is broadcast along its row / column group each step (the only exchange step).

A "step" = one multiply (slicing + pair GEMMs + exact combine) with inputs
resident in HBM; `e2e` = the same through the host-pointer C-ABI call
(H2D of A and B, D2H of C inside the timed region).  Inputs (512 MiB each at
8192^2) exceed the 126 MB L2, so no explicit flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

U53 = 2.0 ** -53

CONFIGS = {
    "c1": dict(name="configs[0]: FP64 GEMM m=n=k=1024, uniform(-0.5,0.5), 4 slices",
               m=1024, n=1024, k=1024, gen="uniform", slices=(4, 4)),
    "c2": dict(name="configs[1]: FP64 GEMM m=n=k=8192, uniform(-0.5,0.5), estimator-chosen "
                    "slices for a 1e-15 target (s=3..8 sweep alongside)",
               m=8192, n=8192, k=8192, gen="uniform", slices="estimator", sweep=(3, 8)),
    "c3": dict(name="configs[2]: badly scaled m=n=k=4096, gen_kappa_d(2^60, seed 7, rotate), "
                    "estimator-chosen slices for 1e-15",
               m=4096, n=4096, k=4096, gen="kappa_d", slices="estimator"),
    "c4": dict(name="configs[3]: tall-skinny m=65536, n=k=2048, uniform(-0.5,0.5), "
                    "estimator-chosen slices for 1e-15",
               m=65536, n=2048, k=2048, gen="uniform", slices="estimator"),
    "c5": dict(name="configs[4]: FP64 GEMM m=n=k=32768, uniform(-0.5,0.5), estimator-chosen "
                    "slices for 1e-15, 2-D C tiles over the ranks (strong scaling)",
               m=32768, n=32768, k=32768, gen="uniform", slices="estimator", strong=True),
    "ns": dict(name="north star: FP64 GEMM m=n=k=16384, uniform(-0.5,0.5), estimator-chosen "
                    "slices for 1e-15",
               m=16384, n=16384, k=16384, gen="uniform", slices="estimator"),
}

METRIC = "effective FP64-equiv TFLOP/s (2mnk/t) and int8 tensor-pipe % of peak vs slices"


def _peaks():
    """(int8 dense peak TOPS, its sustained twin, HBM GB/s, how) from the
    driver-measured bf16 cuBLAS rates (sm_100 int8 dense = 2x bf16 per clock)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        bf16 = float(mp["bf16_tflops"])
        sus = float(mp.get("bf16_tflops_sustained", bf16))
        return 2.0 * bf16, 2.0 * sus, float(mp.get("hbm_gbs", 6535.4)), \
            f"peak = 2 x measured bf16 cuBLAS burst ({bf16} TFLOP/s, MEASURED_PEAKS.json; " \
            f"the conservative choice); peak_sustained = 2 x the sustained bf16 rate ({sus}), " \
            f"the figure for a kernel timed inside a long step.  Unthrottled tcgen05 " \
            f"kind::i8 issue ceiling measured with tools/ubench/mma_rate.cu: 128 cycles per " \
            f"128x256x32 MMA (4.6 POPS at 1965 MHz)"
    except Exception:
        return 2.0 * 1590.0, 2.0 * 1590.0, 6650.0, \
            "2 x fallback bf16 1.59 PFLOP/s (B200_PROFILING.md)"


def _traffic(workload: str):
    path = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def chunk_count(sa, sb, k, t):
    """Chunk planes of the levelled-exact plan (reduced schedule): each
    diagonal's pairs in runs whose int32 sum cannot overflow (build_chunks)."""
    cap = max(1, (2**31 - 1) // (k * (2**t - 1) ** 2))
    dmax = max(sa, sb)
    total = 0
    for d in range(dmax):
        lo, hi = max(1, d + 2 - sb), min(sa, d + 1)
        w = max(0, hi - lo + 1)
        total += -(-w // cap)
    return total


def make_inputs(oz, cfg, rank_i=0, rank_j=0):
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    if cfg["gen"] == "uniform":
        a = oz.random_uniform(m, k, 1 + 1000 * rank_i, -0.5, 0.5)
        b = oz.random_uniform(k, n, 2 + 1000 * rank_j, -0.5, 0.5)
    else:
        a, b = oz.gen_kappa_d(k, 2.0 ** 60, 7 + 1000 * (rank_i + rank_j), True)
    return a, b


def choose_slices(oz, cfg, a, b):
    if cfg["slices"] != "estimator":
        return tuple(cfg["slices"]), None
    mcfg = oz.MmaConfig.int8_int32()
    t = oz.optimal_slice_width(mcfg, cfg["k"])
    prof = oz.scaling_profile(a, b)
    acc_bits = 2 * t + (cfg["k"] - 1).bit_length()
    sel = oz.select_slices(prof.kappa_a, prof.kappa_b, t, U53, 24,
                           oz.SelectOptions(target=1e-15, acc_bits_used=acc_bits))
    return (sel.slices_a, sel.slices_b), {"kappa_a": prof.kappa_a, "kappa_b": prof.kappa_b,
                                          "target": 1e-15, "lhs": sel.lhs}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "power_w_max": max(power), "samples": len(sm), "reasons": sorted(reasons)}


def bad_clocks(c) -> bool:
    r = set(c.get("reasons") or [])
    if r & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}:
        return True
    if c.get("sm_mhz") and c.get("sm_max_mhz") and not r and c["sm_mhz"] < 0.6 * c["sm_max_mhz"]:
        return True
    return False


def cpu_blocks(m, n, count, bs):
    """Deterministic spread of `count` bs x bs C blocks."""
    out = []
    nbr, nbc = max(1, m // bs), max(1, n // bs)
    for t in range(count):
        bi = (t * 7919 + 3) % nbr
        bj = (t * 104729 + 5) % nbc
        out.append((bi * bs, min(m, bi * bs + bs), bj * bs, min(n, bj * bs + bs)))
    return out


def run_cpu_reference(a, b, slices, blocks, threads):
    """Reference multiply() (oracle/_ref) over sampled C blocks -> (C, seconds)."""
    from oracle import pyoracle
    return pyoracle.ref_multiply_blocks(a, b, slices[0], slices[1], blocks, threads)


def reference_arm(args, cfg_key):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2506_11277_b200 as oz  # host-side generator + estimator only
    from oracle import pyoracle
    cfg = CONFIGS[cfg_key]
    line = {"metric": METRIC, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic: reference generator random_uniform(-0.5,0.5) seeds 1,2"
                    if cfg["gen"] == "uniform" else
                    "synthetic: reference gen_kappa_d(2^60, seed 7, rotate)",
            "config": {"workload": cfg["name"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"]}}
    if not pyoracle.have_ref():
        line["unavailable"] = "oracle/_ref/libozref.so not built"
        print(json.dumps(line))
        return
    a, b = make_inputs(oz, cfg)
    try:
        slices, est = choose_slices(oz, cfg, a, b)
    except Exception:
        # no GPU for the estimator's kappa scan: run the reference estimator
        ka, kb, _, _ = pyoracle.ref_scaling_profile(a, b)
        t = 7
        acc = 2 * t + (cfg["k"] - 1).bit_length()
        sel = pyoracle.ref_select_slices(ka, kb, t, U53, 24, target=1e-15, acc_bits_used=acc)
        slices, est = (sel["slices_a"], sel["slices_b"]), {"kappa_a": ka, "kappa_b": kb}
    if cfg["slices"] != "estimator":
        slices = tuple(cfg["slices"])
    threads = os.cpu_count() or 1
    bs = 32 if cfg["k"] >= 4096 else 64
    if cfg["m"] * cfg["n"] <= 1024 * 1024 and cfg["k"] <= 1024:
        bs = 64
    blocks = cpu_blocks(cfg["m"], cfg["n"], threads, bs)
    rates, walls = [], []
    for s in range(args.warmup + args.steps):
        _, secs = run_cpu_reference(a, b, slices, blocks, threads)
        flops = sum(2.0 * (r1 - r0) * (c1 - c0) * cfg["k"] for r0, r1, c0, c1 in blocks)
        if s >= args.warmup:
            rates.append(flops / secs / 1e12)
            walls.append(secs)
    value = statistics.mean(rates)
    sample = (f"{len(blocks)} C blocks of {bs}x{bs} with full k={cfg['k']} per step, reference "
              f"multiply() (oracle/_ref, compiled from the reference sources) on {threads} "
              f"host threads; rate = sampled FP64-equiv flops / wall time")
    line.update({"value": value, "ms_per_step": 1e3 * statistics.mean(walls),
                 "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads,
                                  "kind": "reference", "sample": sample},
                 "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    line["config"].update({"slices": list(slices), "chi": oz.chi(*slices)})
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        reference_arm(args, args.config)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_11277_b200 as oz
    from paper_2506_11277_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["OZGPU_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cfg = dict(CONFIGS[args.config])
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    pr, pc = shard.grid_for(world)
    strong = bool(cfg.get("strong"))
    if strong:
        # a fixed global m x n split into the ranks' C blocks
        blk = shard.block_of(rank, world, m, n)
        gm, gn = m, n
        m, n = blk.row1 - blk.row0, blk.col1 - blk.col0
        cfg["m"], cfg["n"] = m, n
    else:
        # weak scaling: every rank a full m x n block of a (p_r m) x (p_c n) product
        blk = shard.block_of(rank, world, pr * m, pc * n)
        gm, gn = pr * m, pc * n
    mcfg = oz.MmaConfig.int8_int32()
    dev = torch.device(f"cuda:{local}")
    # a dedicated stream: CUDA events and the library's kernels share it
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))

    # inputs: A row-panel i on rank (i, 0), B column-panel j on rank (0, j)
    a_h, b_h = make_inputs(oz, cfg, blk.i, blk.j)
    slices, est = choose_slices(oz, cfg, a_h, b_h)
    if world > 1:  # one plan for the whole job: the max over ranks
        t = torch.tensor(list(slices), device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        slices = tuple(int(v) for v in t.tolist())
    plan = oz.make_plan(mcfg, k, slices[0], slices[1])
    chi = oz.chi(*slices)
    a_d = torch.from_numpy(a_h).to(dev)
    b_d = torch.from_numpy(b_h).to(dev)
    c_d = torch.empty((m, n), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    xchg = shard.PanelExchange(world, rank)

    def step(p=plan):
        xchg.exchange(a_d, b_d)  # A row-panel / B column-panel from their owners (NCCL)
        oz.multiply_device(m, n, k, a_d.data_ptr(), k, b_d.data_ptr(), n, c_d.data_ptr(), n,
                           mcfg, p, stream=torch.cuda.current_stream().cuda_stream,
                           status_ptr=status.data_ptr())

    def timed(nsteps, p=plan):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        stream = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        l0 = oz.kernel_launches()
        e0.record(stream)
        for _ in range(nsteps):
            step(p)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = oz.kernel_launches() - l0
        ms = e0.elapsed_time(e1) / nsteps
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(status.item()) != 0:
        raise RuntimeError("multiply: inputs must be finite with no negative zeros")

    # headline: K steps with nothing else on the stream (after the warm-up the
    # device path replays a captured CUDA graph of the whole multiply)
    sampler = ClockSampler(local)
    attempt = 0
    while True:
        sampler.start()
        ms, launches = timed(args.steps)
        clocks = sampler.stop()
        attempt += 1
        if not bad_clocks(clocks) or attempt >= 2:
            break
    if attempt == 2:
        clocks["remeasured"] = True
    # stage breakdown (CUDA events between the stages; eager launches)
    oz.stage_times(reset=True)
    oz.set_stage_timing(True)
    timed(args.steps)  # as long as the headline loop: the same power-capped clock
    oz.set_stage_timing(False)
    slice_ms, gemm_ms, comb_ms, calls = oz.stage_times(reset=True)

    flops_rank = 2.0 * m * n * k  # this rank's block
    flops_total = 2.0 * gm * gn * k  # the whole job (all ranks' blocks)
    value = flops_total / (ms * 1e-3) / 1e12
    gemm_ms_call = gemm_ms / max(calls, 1)
    int8_ops = 2.0 * chi * m * n * k
    tops = int8_ops / (gemm_ms_call * 1e-3) / 1e12
    peak, peak_sus, hbm_peak, peak_how = _peaks()
    # the driver's rule: the burst peak for a kernel timed alone, the
    # sustained (power-capped) one for a kernel timed inside a long step
    long_region = ms * args.steps >= 500.0
    peak_used = peak_sus if long_region else peak
    peak_kind = ("of measured: 2 x bf16 cuBLAS sustained (timed region %.0f ms >= 500 ms)" if
                 long_region else "of measured: 2 x bf16 cuBLAS burst (timed region %.0f ms)") % \
        (ms * args.steps)
    slice_bytes = 8.0 * (m * k + k * n) + slices[0] * m * k + slices[1] * k * n + 4.0 * (m + n)
    nch = chunk_count(slices[0], slices[1], k, plan.width)
    comb_bytes = 4.0 * nch * m * n + 8.0 * m * n + 4.0 * (m + n)
    slice_ms_call = slice_ms / max(calls, 1)

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "int8",
        "data": "synthetic: reference generator random_uniform(-0.5,0.5) seeds 1,2 "
                "(per-panel seeds 1+1000i / 2+1000j for N>1)" if cfg["gen"] == "uniform" else
                "synthetic: reference gen_kappa_d(2^60, seed 7, rotate)",
        "config": {"workload": cfg["name"], "m": m, "n": n, "k": k,
                   "global_m": gm, "global_n": gn, "grid": [pr, pc],
                   "slices": list(slices), "chi": chi, "width": plan.width,
                   "schedule": "reduced", "strategy": "levelled-exact", "estimator": est,
                   "launch": "CUDA-graph replay of the whole multiply (captured on the 2nd call); "
                             "stage_ms / int8_tops from a second loop of the same length, eager, "
                             "with CUDA events between the stages",
                   "l2": "inputs larger than L2 (A, B = %d MiB each > 126 MB)" %
                         (8 * m * k // 2**20), "parallelism": f"2-D C tiles {pr}x{pc}"},
        "int8_tops": tops,
        "stage_ms": {"slicing": slice_ms_call, "pair_gemms": gemm_ms_call,
                     "combine": comb_ms / max(calls, 1)},
        "roofline": {"bound": "tensor", "achieved": tops, "peak": peak_used, "unit": "TFLOP/s",
                     "frac": tops / peak_used, "traffic": _traffic(args.config),
                     "peak_kind": peak_kind, "peak_burst": peak, "peak_sustained": peak_sus,
                     "kernel": "gemm_i8_pair_kernel<6> (tcgen05.mma.cta_group::2.kind::i8, "
                               "256x256 tiles, equal-length chunk bins, wave lockstep)",
                     "algorithmic": "2*chi*m*n*k int8 ops per launch", "peak_note": peak_how},
        "slicing_roofline": {"bound": "hbm", "achieved": slice_bytes / (slice_ms_call * 1e-3) / 1e9,
                             "peak": hbm_peak, "unit": "GB/s",
                             "frac": slice_bytes / (slice_ms_call * 1e-3) / 1e9 / hbm_peak,
                             "algorithmic": "8(mk+kn) + s_A mk + s_B kn + 4(m+n) bytes"},
        "combine_roofline": {"bound": "hbm", "achieved": comb_bytes / (comb_ms / max(calls, 1) * 1e-3) / 1e9,
                             "peak": hbm_peak, "unit": "GB/s",
                             "frac": comb_bytes / (comb_ms / max(calls, 1) * 1e-3) / 1e9 / hbm_peak,
                             "algorithmic": "4 * chunks * m * n (int32 chunk planes) + 8 m n (C) bytes",
                             "chunks": nch},
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks,
    }

    # s = 3..8 sweep of configs[1] (same inputs), fewer steps each
    if cfg.get("sweep") and not args.no_sweep:
        sweep = []
        for s in range(cfg["sweep"][0], cfg["sweep"][1] + 1):
            ps = oz.make_plan(mcfg, k, s, s)
            for _ in range(2):
                step(ps)
            oz.stage_times(reset=True)
            oz.set_stage_timing(True)
            sms, _ = timed(max(3, args.steps // 4), ps)
            oz.set_stage_timing(False)
            _, g_ms, _, c_ = oz.stage_times(reset=True)
            ch = oz.chi(s, s)
            sweep.append({"s": s, "chi": ch, "tflops": flops_total / (sms * 1e-3) / 1e12,
                          "int8_tops": 2.0 * ch * m * n * k / (g_ms / max(c_, 1) * 1e-3) / 1e12,
                          "ms_per_step": sms})
        line["sweep"] = sweep

    # context only (off the product path): cuBLAS DGEMM on the same device
    # operands, the native FP64 rate the emulation is compared with
    # (PAPER.md:548 reports 7.6x over it at s=3 on B200)
    if world == 1 and not args.no_sweep:
        try:
            ad, bd = a_d[:m, :k], b_d[:k, :n]
            torch.matmul(ad, bd)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                torch.matmul(ad, bd)
            e1.record()
            torch.cuda.synchronize()
            dms = e0.elapsed_time(e1) / reps
            line["fp64_dgemm_reference"] = {
                "api": "torch.matmul float64 (cuBLAS DGEMM), same inputs, not on the product path",
                "tflops": flops_rank / (dms * 1e-3) / 1e12, "ms": dms,
                "speedup_estimator_slices": (flops_rank / (ms * 1e-3) / 1e12) /
                                            (flops_rank / (dms * 1e-3) / 1e12),
                "speedup_s3": (line["sweep"][0]["tflops"] / world) /
                              (flops_rank / (dms * 1e-3) / 1e12) if line.get("sweep") else None}
        except Exception as e:  # context only: never fail the bench line
            line["fp64_dgemm_reference"] = {"error": repr(e)}

    # e2e through the host-pointer C-ABI call (pinned host buffers)
    if not args.no_e2e:
        a_p = torch.from_numpy(a_h).pin_memory().numpy()
        b_p = torch.from_numpy(b_h).pin_memory().numpy()
        c_p = torch.empty((m, n), dtype=torch.float64).pin_memory().numpy()
        oz.multiply(a_p, b_p, mcfg, plan, out=c_p)
        e2e_steps = max(3, args.steps // 4)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            oz.multiply(a_p, b_p, mcfg, plan, out=c_p)
        el = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        line["e2e"] = {"value": flops_total / el / 1e12, "unit": "TFLOP/s",
                       "h2d_bytes_per_step": 8 * (m * k + k * n), "d2h_bytes_per_step": 8 * m * n,
                       "ms_per_step": el * 1e3, "api": "ozgpu_dgemm (host pointers, pinned)"}

    # CPU baseline: the reference itself on sampled blocks, rank 0 at N=1 only
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle import pyoracle
            if pyoracle.have_ref():
                threads = os.cpu_count() or 1
                bs = 64
                blocks = cpu_blocks(m, n, threads, bs)
                c_ref, secs = run_cpu_reference(a_h, b_h, slices, blocks, threads)
                step(plan)  # C of the headline plan (the sweep overwrote c_d)
                torch.cuda.synchronize()
                c_gpu = c_d.cpu().numpy()
                same = all(np.array_equal(c_ref[r0:r1, c0:c1].view(np.uint64),
                                          c_gpu[r0:r1, c0:c1].view(np.uint64))
                           for r0, r1, c0, c1 in blocks)
                flops = sum(2.0 * (r1 - r0) * (c1 - c0) * k for r0, r1, c0, c1 in blocks)
                line["cpu_baseline"] = {
                    "value": flops / secs / 1e12, "unit": "TFLOP/s", "cores": threads,
                    "kind": "reference",
                    "sample": f"{len(blocks)} C blocks of {bs}x{bs} with full k={k}, reference "
                              f"multiply() (oracle/_ref) one std::thread per block; "
                              f"{secs:.1f} s; rate extrapolates to the full product",
                    "blocks_bit_exact_vs_gpu": bool(same)}
            else:
                line["cpu_baseline"] = None
        except Exception as e:  # never let the baseline break the GPU line
            line["cpu_baseline"] = {"error": repr(e)}

    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

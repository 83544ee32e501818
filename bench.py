#!/usr/bin/env python3
"""Benchmark of the B200-native Ozaki-I FP64 GEMM (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Metric (BASELINE.json): effective FP64-equivalent TFLOP/s = 2mnk / t, with
the int8 tensor-pipe rate of the pair GEMMs (2*chi*mnk / t_gemm) reported
against the int8 dense peak as the roofline.

Workload at N=1 (default): configs[1] -- FP64 GEMM m=n=k=8192, uniform(-0.5,
0.5) inputs from the reference generator (seeds 1 and 2), slice counts chosen
by the reference's estimator for a 1e-15 target -> (12, 12),
chi=78; the s=3..8 sweep of the same config and a north-star sub-record
(16384^3, estimator (13, 12)) are reported beside it.

N > 1 (default configs[4]): strong scaling of the 32768^3 product over 2-D C
tiles, one process per GPU over NCCL.  Rank (i, j) computes its C block with
the full k; A row-panel i exists only on rank (i, 0) and B column-panel j only
on rank (0, j) and is broadcast along its row / column group every step (the
only exchange; scales are per row / column so blocks are independent).
Without WORLD_SIZE in the environment, `--gpus N` re-launches itself under
torch.distributed.run with N ranks.  A weak-scaling sub-record (an 8192^3
block per rank) rides along.

A "step" = one multiply (slicing + pair GEMMs + exact combine) with inputs
resident in HBM; `e2e` = the same through the host-pointer C-ABI call
(H2D of A and B, D2H of C inside the timed region, pinned buffers;
`e2e_pageable` from plain pageable arrays).  Inputs (512 MiB each at 8192^2)
exceed the 126 MB L2, so no explicit flush is needed.

`--impl reference` runs the reference's own multiply() (oracle/_ref, compiled
from the unmodified reference sources) on sampled C blocks on all host
cores, with inputs from the reference's generators and slices from the
reference's estimator -- nothing from this repository's package is imported.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
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
    # test-only: the multi-rank code path at a size two ranks can share one GPU with
    "t2": dict(name="test: FP64 GEMM m=n=k=4096, uniform(-0.5,0.5), estimator-chosen slices, "
                    "2-D C tiles over the ranks (strong scaling)",
               m=4096, n=4096, k=4096, gen="uniform", slices="estimator", strong=True),
}

METRIC = "effective FP64-equiv TFLOP/s (2mnk/t) and int8 tensor-pipe % of peak vs slices"


def _load_shard():
    """paper_2506_11277_b200/shard.py as a standalone module (pure Python; the
    package itself, which loads the CUDA library, is not imported)."""
    path = os.path.join(ROOT, "paper_2506_11277_b200", "shard.py")
    spec = importlib.util.spec_from_file_location("_oz_shard", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


shard = _load_shard()


# ------------------------------------------------------------ plan facts
# (host arithmetic shared by both arms so their config records are identical)

def ceil_log2(x: int) -> int:
    return (x - 1).bit_length()


def slice_width(k: int) -> int:
    """optimal_slice_width (mma_sim.cpp:50-59) for MmaConfig::int8_int32()."""
    return min(7, (31 - ceil_log2(k)) // 2)


def chi_of(sa: int, sb: int) -> int:
    """chi (scheme.cpp:46-52), the reduced schedule's pair count."""
    lo, hi = min(sa, sb), max(sa, sb)
    return lo * (2 * hi - lo + 1) // 2


def chunk_count(sa, sb, k, t):
    """Chunk planes of the levelled-exact plan (reduced schedule): each
    diagonal's pairs in runs whose int32 sum cannot overflow (build_chunks)."""
    cap = max(1, (2**31 - 1) // (k * (2**t - 1) ** 2))
    total = 0
    for d in range(max(sa, sb)):
        lo, hi = max(1, d + 2 - sb), min(sa, d + 1)
        total += -(-max(0, hi - lo + 1) // cap)
    return total


def sample_block(k: int) -> int:
    """Edge of the sampled C blocks the CPU legs time (one block per core): a
    block costs ~b^2 k chi int8 MACs on the reference's scalar loop, so b
    shrinks with k to keep one sample step at a few seconds."""
    return 64 if k <= 2048 else 32 if k <= 8192 else 16


def cpu_blocks(m, n, count, bs):
    """Deterministic spread of `count` bs x bs C blocks."""
    out = []
    nbr, nbc = max(1, m // bs), max(1, n // bs)
    for t in range(count):
        bi = (t * 7919 + 3) % nbr
        bj = (t * 104729 + 5) % nbc
        out.append((bi * bs, min(m, bi * bs + bs), bj * bs, min(n, bj * bs + bs)))
    return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def geometry(cfg, world, rank):
    """(block, m, n, global_m, global_n): strong scaling splits the configured
    product; weak scaling gives every rank a full configured-size block."""
    pr, pc = shard.grid_for(world)
    if cfg.get("strong"):
        gm, gn = cfg["m"], cfg["n"]
    else:
        gm, gn = pr * cfg["m"], pc * cfg["n"]
    blk = shard.block_of(rank, world, gm, gn)
    return blk, blk.row1 - blk.row0, blk.col1 - blk.col0, gm, gn


def config_record(cfg, world, m, n, gm, gn, slices):
    k = cfg["k"]
    pr, pc = shard.grid_for(world)
    return {"workload": cfg["name"], "m": m, "n": n, "k": k, "global_m": gm, "global_n": gn,
            "grid": [pr, pc], "slices": list(slices), "chi": chi_of(*slices),
            "width": slice_width(k), "schedule": "reduced", "strategy": "levelled-exact",
            "l2": "inputs larger than L2 (A = %d MiB > 126 MB)" % (8 * m * k // 2**20)
                  if 8 * m * k > 126e6 else "A = %d MiB: operands fit the 126 MB L2 (no flush; launch-bound config)" %
                  (8 * m * k // 2**20),
            "parallelism": f"2-D C tiles {pr}x{pc}"}


def data_note(cfg):
    if cfg["gen"] == "uniform":
        return ("synthetic: reference generator random_uniform(-0.5,0.5), A row-panel i seed "
                "1+1000i, B column-panel j seed 2+1000j (seeds 1, 2 at N=1)")
    return "synthetic: reference gen_kappa_d(2^60, seed 7, rotate)"


def panel_seeds(i, j):
    return 1 + 1000 * i, 2 + 1000 * j


# ------------------------------------------------------------ reference arm

def reference_arm(args, cfg_key):
    """The reference's own CPU path: oracle/_ref is the unmodified reference
    compiled from its sources; inputs from its generators, slices from its
    estimator (scaling_profile + select_slices); nothing from the product."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import pyoracle as po
    cfg = CONFIGS[cfg_key]
    blk, m, n, gm, gn = geometry(cfg, world, 0)
    k = cfg["k"]
    line = {"metric": METRIC, "unit": "TFLOP/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
            "dtype": "int8", "data": data_note(cfg)}
    if not po.have_ref():
        line["unavailable"] = "oracle/_ref/libozref.so not built"
        print(json.dumps(line))
        return
    if cfg["gen"] == "uniform":
        sa_, sb_ = panel_seeds(blk.i, blk.j)
        a = po.ref_random_uniform(m, k, sa_, -0.5, 0.5)
        b = po.ref_random_uniform(k, n, sb_, -0.5, 0.5)
    else:
        a, b = po.ref_gen_kappa_d(k, 2.0 ** 60, 7, True)
    t = slice_width(k)
    if cfg["slices"] == "estimator":
        ka, kb, _, _ = po.ref_scaling_profile(a, b)
        sel = po.ref_select_slices(ka, kb, t, U53, 24, target=1e-15,
                                   acc_bits_used=2 * t + ceil_log2(k))
        slices = (sel["slices_a"], sel["slices_b"])
        est = {"kappa_a": ka, "kappa_b": kb, "target": 1e-15, "lhs": sel["lhs"],
               "via": "reference scaling_profile + select_slices (analysis.cpp:58-68,142-207)"}
    else:
        slices, est = tuple(cfg["slices"]), None
    threads = os.cpu_count() or 1
    bs = sample_block(k)
    blocks = cpu_blocks(m, n, threads, bs)
    rates, walls = [], []
    for s in range(args.warmup + args.steps):
        _, secs = po.ref_multiply_blocks(a, b, slices[0], slices[1], blocks, threads)
        flops = sum(2.0 * (r1 - r0) * (c1 - c0) * k for r0, r1, c0, c1 in blocks)
        if s >= args.warmup:
            rates.append(flops / secs / 1e12)
            walls.append(secs)
    value = statistics.mean(rates)
    sample = (f"{len(blocks)} C blocks of {bs}x{bs} with full k={k} per step (one per host "
              f"thread), reference multiply() (oracle/_ref, compiled from the reference "
              f"sources) on {threads} threads of {cpu_model()}; rate = sampled FP64-equiv "
              f"flops / wall time (extrapolates to the full product: blocking is exact)")
    line.update({"value": value, "ms_per_step": 1e3 * statistics.mean(walls),
                 "config": config_record(cfg, world, m, n, gm, gn, slices),
                 "estimator": est,
                 "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads,
                                  "kind": "reference", "sample": sample,
                                  "cpu_model": cpu_model(), "nproc": os.cpu_count()},
                 "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line))


# ------------------------------------------------------------ measurement helpers

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


# tcgen05 kind::i8 issue rate per SM: one 128x256x32 MMA (2*128*256*32 ops)
# per 128 cycles (tools/ubench/mma_rate.cu)
I8_OPS_PER_CLK_SM = 2 * 128 * 256 * 32 // 128


def _peaks():
    """(int8 dense peak, its sustained twin, HBM GB/s, how) from the
    driver-measured bf16 cuBLAS rates (sm_100 int8 dense = 2x bf16 per clock)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        bf16 = float(mp["bf16_tflops"])
        sus = float(mp.get("bf16_tflops_sustained", bf16))
        return 2.0 * bf16, 2.0 * sus, float(mp.get("hbm_gbs", 6548.2)), \
            f"peak = 2 x measured bf16 cuBLAS burst ({bf16} TFLOP/s, MEASURED_PEAKS.json): the " \
            f"recipe's figure for a kernel timed inside a short step; frac_sustained uses " \
            f"2 x the sustained bf16 rate ({sus}).  Unthrottled tcgen05 kind::i8 issue " \
            f"ceiling measured with tools/ubench/mma_rate.cu: 128 cycles per 128x256x32 MMA " \
            f"(4.6 POPS at 1965 MHz)"
    except Exception:
        return 2.0 * 1590.0, 2.0 * 1590.0, 6650.0, \
            "2 x fallback bf16 1.59 PFLOP/s (B200_PROFILING.md)"


def _committed_traffic(cfg_key):
    path = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(cfg_key)
    except Exception:
        return None


def measure_traffic(cfg_key, timeout=300):
    """DRAM bytes of one pair-GEMM launch, measured now: this script re-run
    under ncu (dram__bytes_read.sum + dram__bytes_write.sum of the 2nd
    gemm_i8 launch, --clock-control none).  Nothing from that child run is
    used but the counter."""
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{cfg_key}_{os.getpid()}.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--print-units", "base", "-k", "regex:gemm_i8", "-s", "1",
           "-c", "1", "--csv", "--log-file", log, sys.executable, os.path.abspath(__file__),
           "--config", cfg_key, "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
           "--no-sweep", "--no-traffic", "--no-north-star"]
    env = dict(os.environ, OZGPU_GRAPH="0")
    try:
        subprocess.run(cmd, env=env, timeout=timeout, stdout=subprocess.DEVNULL,
                       stderr=subprocess.DEVNULL, cwd=ROOT)
        import csv
        vals, kernel = {}, None
        with open(log) as f:
            rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
        head = rows[0]
        for r in rows[1:]:
            rec = dict(zip(head, r))
            vals[rec["Metric Name"]] = float(rec["Metric Value"].replace(",", ""))
            kernel = rec.get("Kernel Name")
        return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                "read": vals["dram__bytes_read.sum"], "write": vals["dram__bytes_write.sum"],
                "ncu_ns": vals.get("gpu__time_duration.sum"), "kernel": kernel,
                "source": "measured in this run (ncu child, one launch)"}
    except Exception as e:  # context only: never fail the bench line
        c = _committed_traffic(cfg_key)
        return {"bytes": c, "source": f"profiles/ncu_gemm_traffic.json (measurement failed: "
                                      f"{type(e).__name__})"} if c else None
    finally:
        try:
            os.remove(log)
        except OSError:
            pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ------------------------------------------------------------ our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 (configs[1]) at N=1, c5 (configs[4], strong) at N>1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-traffic", action="store_true")
    ap.add_argument("--no-north-star", action="store_true")
    # testing the N>1 path on a single GPU: every rank on cuda:0, gloo collectives
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--same-device", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    env_world = os.environ.get("WORLD_SIZE")
    if args.config is None:
        args.config = "c2" if int(env_world or args.gpus) == 1 else "c5"
    if args.impl == "reference":
        reference_arm(args, args.config)
        return
    if env_world is None and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd, env=dict(os.environ)))
    world = int(env_world or "1")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) in the log

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_11277_b200 as oz

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    os.environ["OZGPU_DEVICE"] = str(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group("gloo")
    cfg = dict(CONFIGS[args.config])
    k = cfg["k"]
    blk, m, n, gm, gn = geometry(cfg, world, rank)
    mcfg = oz.MmaConfig.int8_int32()
    dev = torch.device(f"cuda:{local}")
    # a dedicated stream: CUDA events and the library's kernels share it
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    xchg = shard.PanelExchange(world, rank)

    def load_panels(cfg_):
        """A row-panel i exists only on rank (i, 0), B column-panel j only on
        (0, j); the others receive them in the exchange."""
        blk_, m_, n_, _, _ = geometry(cfg_, world, rank)
        k_ = cfg_["k"]
        a_d = torch.zeros((m_, k_), dtype=torch.float64, device=dev)
        b_d = torch.zeros((k_, n_), dtype=torch.float64, device=dev)
        if cfg_["gen"] == "uniform":
            sa_, sb_ = panel_seeds(blk_.i, blk_.j)
            if rank == shard.a_owner(world, blk_.i):
                a_d.copy_(torch.from_numpy(oz.random_uniform(m_, k_, sa_, -0.5, 0.5)))
            if rank == shard.b_owner(world, blk_.j):
                b_d.copy_(torch.from_numpy(oz.random_uniform(k_, n_, sb_, -0.5, 0.5)))
        else:
            a_h, b_h = oz.gen_kappa_d(k_, 2.0 ** 60, 7, True)
            a_d.copy_(torch.from_numpy(a_h))
            b_d.copy_(torch.from_numpy(b_h))
        xchg.exchange(a_d, b_d)
        torch.cuda.synchronize()
        return a_d, b_d, m_, n_

    def estimate(cfg_, a_h, b_h):
        if cfg_["slices"] != "estimator":
            return tuple(cfg_["slices"]), None
        t = oz.optimal_slice_width(mcfg, cfg_["k"])
        prof = oz.scaling_profile(a_h, b_h)  # the GPU kappa scan
        sel = oz.select_slices(prof.kappa_a, prof.kappa_b, t, U53, 24,
                               oz.SelectOptions(target=1e-15,
                                                acc_bits_used=2 * t + ceil_log2(cfg_["k"])))
        sl = (sel.slices_a, sel.slices_b)
        if world > 1:  # one plan for the whole job: the max over ranks
            tt = torch.tensor(list(sl), device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sl = tuple(int(v) for v in tt.tolist())
        return sl, {"kappa_a": prof.kappa_a, "kappa_b": prof.kappa_b, "target": 1e-15,
                    "lhs": sel.lhs, "via": "GPU kappa scan + host select_slices"}

    a_d, b_d, m, n = load_panels(cfg)
    a_h, b_h = a_d.cpu().numpy(), b_d.cpu().numpy()
    slices, est = estimate(cfg, a_h, b_h)
    plan = oz.make_plan(mcfg, k, slices[0], slices[1])
    chi = oz.chi(*slices)
    c_d = torch.empty((m, n), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)

    def make_step(a_, b_, c_, m_, n_, k_, exchange=True):
        def step(p):
            if exchange:
                xchg.exchange(a_, b_)  # panels from their owners (NCCL broadcast)
            oz.multiply_device(m_, n_, k_, a_.data_ptr(), k_, b_.data_ptr(), n_, c_.data_ptr(), n_,
                               mcfg, p, stream=torch.cuda.current_stream().cuda_stream,
                               status_ptr=status.data_ptr())
        return step

    step = make_step(a_d, b_d, c_d, m, n, k)

    def timed(nsteps, p, stepf=None):
        stepf = stepf or step
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        stream = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        l0 = oz.kernel_launches()
        e0.record(stream)
        for _ in range(nsteps):
            stepf(p)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = oz.kernel_launches() - l0
        ms = e0.elapsed_time(e1) / nsteps
        if world > 1:
            tt = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
            dist.barrier()
        return ms, launches

    for _ in range(args.warmup):
        step(plan)
    torch.cuda.synchronize()
    if int(status.item()) != 0:
        raise RuntimeError("multiply: inputs must be finite with no negative zeros")

    # headline: K steps with nothing else on the stream (after the warm-up the
    # device path replays a captured CUDA graph of the whole multiply)
    sampler = ClockSampler(local)
    attempt = 0
    while True:
        sampler.start()
        ms, launches = timed(args.steps, plan)
        clocks = sampler.stop()
        attempt += 1
        if not bad_clocks(clocks) or attempt >= 2:
            break
    if attempt == 2:
        clocks["remeasured"] = True

    def stage_split(nsteps, p, stepf=None):
        """Stage times from an eager loop of the same length (CUDA events
        between the stages, on the launching stream)."""
        oz.stage_times(reset=True)
        oz.set_stage_timing(True)
        timed(nsteps, p, stepf)
        oz.set_stage_timing(False)
        s_ms, g_ms, c_ms, calls = oz.stage_times(reset=True)
        calls = max(calls, 1)
        return s_ms / calls, g_ms / calls, c_ms / calls

    slice_ms, gemm_ms, comb_ms = stage_split(args.steps, plan)
    peak, peak_sus, hbm_peak, peak_how = _peaks()

    def rooflines(m_, n_, k_, sl, g_ms, s_ms, c_ms):
        ch = chi_of(*sl)
        tops = 2.0 * ch * m_ * n_ * k_ / (g_ms * 1e-3) / 1e12
        sbytes = 8.0 * (m_ * k_ + k_ * n_) + sl[0] * m_ * k_ + sl[1] * k_ * n_ + 4.0 * (m_ + n_)
        nch = chunk_count(sl[0], sl[1], k_, slice_width(k_))
        cbytes = 4.0 * nch * m_ * n_ + 8.0 * m_ * n_ + 4.0 * (m_ + n_)
        return tops, {
            "roofline": {"bound": "tensor", "achieved": tops, "peak": peak, "unit": "TFLOP/s",
                         "frac": tops / peak, "traffic": None,
                         "peak_kind": "measured: 2 x bf16 cuBLAS burst (MEASURED_PEAKS.json)",
                         "frac_sustained": tops / peak_sus, "peak_sustained": peak_sus,
                         "kernel": "gemm_i8_pair_kernel (tcgen05.mma.cta_group::2.kind::i8; "
                                   "256x512 tiles when they fill the SMs, else 256x256; "
                                   "equal-length chunk bins, wave lockstep, split-k tail)",
                         "algorithmic": "2*chi*m*n*k int8 ops per launch (%.4g)" %
                                        (2.0 * ch * m_ * n_ * k_),
                         "launch_ms": g_ms, "peak_note": peak_how},
            "slicing_roofline": {"bound": "hbm", "achieved": sbytes / (s_ms * 1e-3) / 1e9,
                                 "peak": hbm_peak, "unit": "GB/s",
                                 "frac": sbytes / (s_ms * 1e-3) / 1e9 / hbm_peak,
                                 "algorithmic": "8(mk+kn) + s_A mk + s_B kn + 4(m+n) bytes "
                                                "(%.4g)" % sbytes, "ms": s_ms},
            "combine_roofline": ({"bound": "hbm", "achieved": cbytes / (c_ms * 1e-3) / 1e9,
                                  "peak": hbm_peak, "unit": "GB/s",
                                  "frac": cbytes / (c_ms * 1e-3) / 1e9 / hbm_peak,
                                  "algorithmic": "4 * chunks * m * n (int32 chunk planes) + 8 m n "
                                                 "(C) bytes (%.4g)" % cbytes,
                                  "chunks": nch, "ms": c_ms} if c_ms > 0.05 * s_ms else
                                 {"note": "GEMM + combine run over row blocks of C under the "
                                          "chunk-plane budget: the combine time is inside "
                                          "pair_gemms", "chunks": nch, "ms": c_ms})}

    flops_rank = 2.0 * m * n * k  # this rank's block
    flops_total = 2.0 * gm * gn * k  # the whole job (all ranks' blocks)
    value = flops_total / (ms * 1e-3) / 1e12
    tops, roofs = rooflines(m, n, k, slices, gemm_ms, slice_ms, comb_ms)

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak",
        "vs_baseline": None, "dtype": "int8", "data": data_note(cfg),
        "config": config_record(cfg, world, m, n, gm, gn, slices),
        "estimator": est,
        "launch": "headline: CUDA-graph replay of the whole multiply (captured on the 2nd call); "
                  "stage_ms / int8_tops from a second loop of the same length, eager, with "
                  "CUDA events between the stages",
        "int8_tops": tops,
        "stage_ms": {"slicing": slice_ms, "pair_gemms": gemm_ms, "combine": comb_ms},
        **roofs,
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks,
    }
    if clocks.get("sm_mhz"):
        # the tensor pipe's own limit at the clock the run actually held: a
        # power-capped long step runs well below max clock, a short unthrottled
        # one above the cuBLAS-derived burst figure (frac > 1 there)
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        pk = I8_OPS_PER_CLK_SM * nsm * clocks["sm_mhz"] * 1e6 / 1e12
        line["roofline"].update({
            "peak_at_clock": pk, "frac_at_clock": tops / pk,
            "peak_at_clock_note": "%d SMs x %d int8 ops/clk/SM (one 128x256x32 kind::i8 MMA "
                                  "per 128 cycles per SM, tools/ubench/mma_rate.cu) x the "
                                  "median SM clock of the timed region (%d MHz)" %
                                  (nsm, I8_OPS_PER_CLK_SM, clocks["sm_mhz"])})
    if world > 1:
        line["exchange"] = ("A row-panel (%d x %d) broadcast along row groups, B column-panel "
                            "(%d x %d) along column groups (NCCL), inside every timed step" %
                            (m, k, k, n))

    # s = 3..8 sweep of configs[1] (same inputs), fewer steps each
    if cfg.get("sweep") and not args.no_sweep:
        sweep = []
        for s in range(cfg["sweep"][0], cfg["sweep"][1] + 1):
            ps = oz.make_plan(mcfg, k, s, s)
            for _ in range(2):
                step(ps)
            sms, _ = timed(max(3, args.steps // 4), ps)
            _, g_ms, _ = stage_split(max(3, args.steps // 4), ps)
            ch = oz.chi(s, s)
            sweep.append({"s": s, "chi": ch, "tflops": flops_total / (sms * 1e-3) / 1e12,
                          "int8_tops": 2.0 * ch * m * n * k / (g_ms * 1e-3) / 1e12,
                          "ms_per_step": sms})
        line["sweep"] = sweep

    # context only (off the product path): cuBLAS DGEMM on the same device
    # operands, the native FP64 rate the emulation is compared with
    # (PAPER.md:548 reports 7.6x over it at s=3 on B200)
    if world == 1 and not args.no_sweep:
        try:
            torch.matmul(a_d, b_d)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                torch.matmul(a_d, b_d)
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

    # accuracy beside the speed (the other half of "vs slices"): forward
    # error of every sweep point, of the estimator's choice and of cuBLAS
    # DGEMM against RN(AB) from oz.exact_gemm (error-free slices, bitwise the
    # reference's GMP exact_gemm); PAPER.md:548-550 puts DGEMM-equivalent
    # accuracy at s = 7 for uniform inputs
    if world == 1 and cfg.get("sweep") and not args.no_sweep:
        try:
            exact = torch.from_numpy(oz.exact_gemm(a_h, b_h)).to(dev)
            e_norm = torch.linalg.norm(exact)
            tiny = torch.finfo(torch.float64).tiny

            def errs(cd):
                diff = cd - exact
                return {"max_rel": float((diff.abs() / exact.abs().clamp_min(tiny)).max()),
                        "frobenius_rel": float(torch.linalg.norm(diff) / e_norm)}

            acc = {"reference": "RN(AB) from oz.exact_gemm", "by_slices": {}}
            for sv in range(cfg["sweep"][0], cfg["sweep"][1] + 1):
                step(oz.make_plan(mcfg, k, sv, sv))
                torch.cuda.synchronize()
                acc["by_slices"][str(sv)] = errs(c_d)
            step(plan)
            torch.cuda.synchronize()
            acc["estimator_slices"] = {"slices": list(slices), **errs(c_d)}
            acc["cublas_dgemm"] = errs(torch.matmul(a_d, b_d))
            line["accuracy"] = acc
            del exact
        except Exception as e:  # context only: never fail the bench line
            line["accuracy"] = {"error": repr(e)}

    # e2e through the host-pointer C-ABI call: pinned buffers (the contract),
    # and plain pageable arrays (what std::vector / numpy callers pass)
    if not args.no_e2e:
        def e2e_run(a_src, b_src, c_dst, nsteps):
            oz.multiply(a_src, b_src, mcfg, plan, out=c_dst)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(nsteps):
                oz.multiply(a_src, b_src, mcfg, plan, out=c_dst)
            el = (time.perf_counter() - t0) / nsteps
            if world > 1:
                tt = torch.tensor([el], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                el = float(tt.item())
            return el
        e2e_steps = max(3, args.steps // 4)
        a_p = torch.from_numpy(a_h).pin_memory().numpy()
        b_p = torch.from_numpy(b_h).pin_memory().numpy()
        c_p = torch.empty((m, n), dtype=torch.float64).pin_memory().numpy()
        el = e2e_run(a_p, b_p, c_p, e2e_steps)
        line["e2e"] = {"value": flops_total / el / 1e12, "unit": "TFLOP/s",
                       "h2d_bytes_per_step": 8 * (m * k + k * n), "d2h_bytes_per_step": 8 * m * n,
                       "ms_per_step": el * 1e3,
                       "api": "ozgpu_dgemm (host pointers, pinned buffers), wall clock, max "
                              "over ranks"}
        del a_p, b_p, c_p
        c_pg = np.empty((m, n))
        el = e2e_run(a_h, b_h, c_pg, e2e_steps)
        line["e2e_pageable"] = {"value": flops_total / el / 1e12, "unit": "TFLOP/s",
                                "ms_per_step": el * 1e3,
                                "api": "ozgpu_dgemm (host pointers, pageable numpy arrays)"}
        del c_pg

    # CPU baseline: the reference itself on sampled blocks, rank 0 at N=1 only
    def cpu_sample(a_, b_, sl, k_, m_, n_, c_dev):
        from oracle import pyoracle
        if not pyoracle.have_ref():
            return None
        threads = os.cpu_count() or 1
        bs = sample_block(k_)
        blocks = cpu_blocks(m_, n_, threads, bs)
        c_ref, secs = pyoracle.ref_multiply_blocks(a_, b_, sl[0], sl[1], blocks, threads)
        c_gpu = c_dev.cpu().numpy()
        same = all(np.array_equal(c_ref[r0:r1, c0:c1].view(np.uint64),
                                  c_gpu[r0:r1, c0:c1].view(np.uint64))
                   for r0, r1, c0, c1 in blocks)
        flops = sum(2.0 * (r1 - r0) * (c1 - c0) * k_ for r0, r1, c0, c1 in blocks)
        return {"value": flops / secs / 1e12, "unit": "TFLOP/s", "cores": threads,
                "kind": "reference", "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                "sample": f"{len(blocks)} C blocks of {bs}x{bs} with full k={k_}, reference "
                          f"multiply() (oracle/_ref) one std::thread per block on {threads} "
                          f"threads of {cpu_model()}; {secs:.1f} s; rate extrapolates to the "
                          f"full product (blocking is exact)",
                "blocks_bit_exact_vs_gpu": bool(same), "blocks": len(blocks)}

    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            step(plan)  # C of the headline plan (the sweep overwrote c_d)
            torch.cuda.synchronize()
            line["cpu_baseline"] = cpu_sample(a_h, b_h, slices, k, m, n, c_d)
        except Exception as e:  # never let the baseline break the GPU line
            line["cpu_baseline"] = {"error": repr(e)}

    # DRAM traffic of the pair GEMM, measured now by an ncu child run
    if world == 1 and not args.no_traffic:
        tr = measure_traffic(args.config)
        if tr and tr.get("bytes"):
            line["roofline"]["traffic"] = tr["bytes"]
            line["roofline"]["traffic_detail"] = tr

    # sub-records measured in this same run (so the driver's own bench call
    # carries them): the north star 16384^3, configs[2] (kappa_D 4096^3) and
    # configs[3] (65536 x 2048^2), each at the estimator's slices with its
    # own roofline, clocks and sampled bit-exact CPU-reference blocks
    def sub_record(key, nsteps):
        sc = dict(CONFIGS[key])
        a2, b2, m2, n2 = load_panels(sc)
        a2h, b2h = a2.cpu().numpy(), b2.cpu().numpy()
        sl2, est2 = estimate(sc, a2h, b2h)
        p2 = oz.make_plan(mcfg, sc["k"], *sl2)
        c2 = torch.empty((m2, n2), dtype=torch.float64, device=dev)
        step2 = make_step(a2, b2, c2, m2, n2, sc["k"], exchange=False)
        for _ in range(3):
            step2(p2)
        sampler.start()
        ms2, _ = timed(nsteps, p2, step2)
        clk2 = sampler.stop()
        s2, g2, cc2 = stage_split(nsteps, p2, step2)
        tops2, roofs2 = rooflines(m2, n2, sc["k"], sl2, g2, s2, cc2)
        if clk2.get("sm_mhz"):
            nsm = torch.cuda.get_device_properties(dev).multi_processor_count
            pk = I8_OPS_PER_CLK_SM * nsm * clk2["sm_mhz"] * 1e6 / 1e12
            roofs2["roofline"].update({"peak_at_clock": pk, "frac_at_clock": tops2 / pk})
        rec = {"workload": sc["name"], "slices": list(sl2), "chi": chi_of(*sl2),
               "estimator": est2, "steps": nsteps, "ms_per_step": ms2,
               "value": 2.0 * m2 * n2 * sc["k"] / (ms2 * 1e-3) / 1e12, "unit": "TFLOP/s",
               "int8_tops": tops2, "frac_of_4500_tops_spec": tops2 / 4500.0,
               "stage_ms": {"slicing": s2, "pair_gemms": g2, "combine": cc2},
               **roofs2, "clocks": clk2}
        if not args.no_cpu_baseline:
            step2(p2)
            torch.cuda.synchronize()
            rec["cpu_baseline"] = cpu_sample(a2h, b2h, sl2, sc["k"], m2, n2, c2)
        del a2, b2, c2
        torch.cuda.empty_cache()  # give the next sub-record (or the library) the memory back
        return rec

    if world == 1 and args.config == "c2" and not args.no_north_star:
        try:
            line["north_star"] = sub_record("ns", 3)
        except Exception as e:
            line["north_star"] = {"error": repr(e)}
        others = {}
        # configs[4] on this one GPU too: the N = 1 point of its strong-scaling
        # series (the N > 1 lines run configs[4] sharded), ~40 s
        for key, nsteps in (("c3", 10), ("c4", 6), ("c5", 2)):
            try:
                others[key] = sub_record(key, nsteps)
            except Exception as e:
                others[key] = {"error": repr(e)}
        line["other_configs"] = others

    # weak-scaling sub-record at N > 1: every rank an 8192^3 block (configs[1])
    if world > 1 and args.config in ("c5", "t2"):
        try:
            wc = dict(CONFIGS["c2"])
            aw, bw, mw, nw = load_panels(wc)
            slw, _ = estimate(wc, aw.cpu().numpy(), bw.cpu().numpy())
            pw = oz.make_plan(mcfg, wc["k"], *slw)
            cw = torch.empty((mw, nw), dtype=torch.float64, device=dev)
            stepw = make_step(aw, bw, cw, mw, nw, wc["k"])
            for _ in range(3):
                stepw(pw)
            nsteps = max(3, args.steps // 4)
            msw, _ = timed(nsteps, pw, stepw)
            pr, pc = shard.grid_for(world)
            tot = 2.0 * pr * wc["m"] * pc * wc["n"] * wc["k"]
            line["weak_scaling"] = {"workload": "configs[1] block (8192^3) per rank, panels "
                                                "broadcast from their owners each step",
                                    "slices": list(slw), "ms_per_step": msw,
                                    "value": tot / (msw * 1e-3) / 1e12, "unit": "TFLOP/s",
                                    "global_m": pr * wc["m"], "global_n": pc * wc["n"]}
        except Exception as e:
            line["weak_scaling"] = {"error": repr(e)}

    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

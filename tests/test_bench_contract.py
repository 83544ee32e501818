"""bench.py keeps the driver's JSON contract: one line with the required keys
(our arm on the GPU, the reference arm on the CPU)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle import pyoracle
    if not pyoracle.have_ref():
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"], 600)
    assert REQUIRED <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("configs[0]")


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-sweep",
              "--no-cpu-baseline"], 900)
    assert REQUIRED | {"roofline", "gpu_launches", "clocks"} <= set(d)
    assert d["value"] > 1.0 and d["gpu_launches"] >= 3 * 3
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * (1024 * 1024 * 2)
    assert d["e2e"]["d2h_bytes_per_step"] == 8 * 1024 * 1024


def test_bench_geometry_and_config_records():
    """bench.py's sharding geometry (no GPU): strong scaling (configs[4])
    splits the 32768^2 C over the ranks' 2-D tiles, weak scaling gives every
    rank a full block; config records are identical between the two arms'
    code paths for the same world size."""
    import importlib.util
    import numpy as np
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for world in (1, 2, 4, 8):
        cfg = bench.CONFIGS["c5"]
        cover = np.zeros((8, 8), dtype=int)  # 32768 / 4096 coarse cells
        for rank in range(world):
            blk, m, n, gm, gn = bench.geometry(cfg, world, rank)
            assert (gm, gn) == (32768, 32768) and m * n * world == gm * gn
            cover[blk.row0 // 4096:blk.row1 // 4096, blk.col0 // 4096:blk.col1 // 4096] += 1
        assert (cover == 1).all()
        blk, m, n, gm, gn = bench.geometry(bench.CONFIGS["c2"], world, world - 1)
        pr, pc = bench.shard.grid_for(world)
        assert (m, n, gm, gn) == (8192, 8192, 8192 * pr, 8192 * pc)
        r1 = bench.config_record(cfg, world, m, n, gm, gn, (13, 12))
        r2 = bench.config_record(cfg, world, m, n, gm, gn, (13, 12))
        assert r1 == r2 and r1["chi"] == 90 and r1["grid"] == [pr, pc]
    assert bench.chi_of(12, 12) == 78 and bench.chunk_count(12, 12, 8192, 7) == 12
    assert bench.sample_block(8192) == 32 and bench.slice_width(16384) == 7


@pytest.mark.gpu
def test_multi_rank_bench_path_on_one_gpu():
    """The N > 1 bench path end to end (bench.py re-launches itself under
    torch.distributed.run, panels exist only on their owner ranks and are
    broadcast every step, max-over-ranks timing, the weak-scaling sub-record)
    with two ranks sharing the one GPU of this run (gloo collectives; the
    NCCL path differs only in the process-group backend)."""
    d = _run(["--gpus", "2", "--config", "t2", "--steps", "3", "--warmup", "3", "--no-sweep",
              "--no-cpu-baseline", "--no-traffic", "--dist-backend", "gloo", "--same-device"],
             900)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["grid"] == [2, 1] and d["config"]["m"] == 2048
    assert "exchange" in d and d["weak_scaling"].get("value", 0) > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * (2048 * 4096 + 4096 * 4096)


@pytest.mark.gpu
def test_headline_line_sub_records():
    """The driver's default config carries the accuracy sweep and the
    north-star / configs[2] / configs[3] / configs[4] sub-records, each
    bit-exact on its sampled CPU-reference blocks."""
    d = _run(["--steps", "3", "--warmup", "3", "--no-e2e", "--no-traffic"], 1500)
    acc = d["accuracy"]
    assert "error" not in acc, acc
    errs = [acc["by_slices"][str(s)]["frobenius_rel"] for s in range(3, 9)]
    assert all(x > y for x, y in zip(errs, errs[1:])), errs  # more slices, smaller error
    assert acc["estimator_slices"]["frobenius_rel"] < acc["cublas_dgemm"]["frobenius_rel"]
    for rec in [d["north_star"], d["other_configs"]["c3"], d["other_configs"]["c4"],
                d["other_configs"]["c5"]]:
        assert "error" not in rec, rec
        assert rec["value"] > 1.0 and rec["roofline"]["achieved"] > 0
        assert rec["cpu_baseline"]["blocks_bit_exact_vs_gpu"] is True
    assert d["other_configs"]["c3"]["slices"] == [16, 17]
    assert d["other_configs"]["c4"]["slices"] == [12, 11]
    assert d["north_star"]["slices"] == [13, 12]
    assert d["other_configs"]["c5"]["slices"] == [13, 12]

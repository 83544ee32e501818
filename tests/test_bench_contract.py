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

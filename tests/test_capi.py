"""The C-ABI library loads and exports every entry point include/ozgpu.h
declares; without a GPU every compute call fails loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import HAS_GPU, ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "ozgpu.h")).read()
    return sorted(set(re.findall(r"\b(ozgpu_[a-z_0-9]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(oz):
    names = _declared()
    assert len(names) >= 24
    lib = ctypes.CDLL(oz.library_path())
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", oz.library_path()], capture_output=True,
                         text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a(oz):
    out = subprocess.run(["cuobjdump", "--list-elf", oz.library_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", oz.library_path()], capture_output=True,
                          text=True).stdout
    # tcgen05 tensor-core MMAs (1-CTA and CTA-pair) and TMA loads are present
    assert "UTCIMMA" in sass and "UTCIMMA.2CTA" in sass and "UTMALDG" in sass
    assert "HMMA" not in sass and "IMMA.16" not in sass  # no legacy mma.sync path


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(oz):
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, 4, 2, 2)
    with pytest.raises(oz.DeviceError):
        oz.multiply(np.ones((3, 4)), np.ones((4, 2)), cfg, plan)
    with pytest.raises(oz.DeviceError):
        oz.split_rows(np.ones((2, 2)), 7, 2)
    with pytest.raises(oz.DeviceError):
        oz.integer_gemm(np.ones((2, 2), dtype=np.int64), np.ones((2, 2), dtype=np.int64), cfg)
    ctx = ctypes.c_void_p()
    lib = ctypes.CDLL(oz.library_path())
    assert lib.ozgpu_create(0, ctypes.byref(ctx)) == 3


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "ozgpu.h"\nint main(void){ozgpu_plan p; (void)p; return 0;}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-c", str(src), "-o", str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_generators_live_outside_the_product_library(oz, ref):
    """random_uniform / gen_kappa_d (the benchmark inputs) come from
    lib/libozgen.so, not libozgpu.so, with the reference generators' bytes."""
    out = subprocess.run(["nm", "-D", "--defined-only", oz.library_path()], capture_output=True,
                         text=True).stdout
    assert "random_uniform" not in out and "kappa_d" not in out
    a = oz.random_uniform(33, 17, 5, -0.5, 0.5)
    assert np.array_equal(a.view(np.uint64), ref.ref_random_uniform(33, 17, 5, -0.5, 0.5).view(np.uint64))
    x, y = oz.gen_kappa_d(40, 2.0 ** 60, 7, True)
    wx, wy = ref.ref_gen_kappa_d(40, 2.0 ** 60, 7, True)
    assert np.array_equal(x.view(np.uint64), wx.view(np.uint64))
    assert np.array_equal(y.view(np.uint64), wy.view(np.uint64))

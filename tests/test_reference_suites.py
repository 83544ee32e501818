"""The reference's own test suites (proj/tests/*_test.cpp), compiled in place
against the unmodified reference by oracle/Makefile, pass: the oracle we
compare against is the real, healthy reference."""
import os
import subprocess

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "oracle", "_ref")
SUITES = ["fpcore", "slicing", "mma_sim", "scheme", "analysis", "oracle", "generators"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite(ref, suite):
    exe = os.path.join(REF, f"{suite}_test")
    if not os.path.exists(exe):
        pytest.skip("suite not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_reference_acceptance(ref):
    exe = os.path.join(REF, "acceptance_test")
    if not os.path.exists(exe):
        pytest.skip("acceptance suite not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:]
    assert r.stdout.count("[PASS]") == 9

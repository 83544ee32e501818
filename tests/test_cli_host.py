"""The reference's cli_test cases that need no GPU, run against this repo's
`ozmul` binary (the matrix-file round trip and reader errors, the sweep
grammar, the I/O exit code, the capacity check that fails before any GPU
work), plus the binary's usage contract."""
import os
import subprocess

import pytest

from conftest import ROOT
from test_conformance import CLI_HOST_CASES, _cli_case

CLI = os.path.join(ROOT, "paper_2506_11277_b200", "lib", "ozmul")


@pytest.mark.parametrize("case", CLI_HOST_CASES)
def test_reference_cli_case_host(case):
    _cli_case(case)


def test_cli_usage_and_exit_codes(tmp_path):
    import __graft_entry__
    __graft_entry__.build_library()
    __graft_entry__.build_cli()
    assert subprocess.run([CLI], capture_output=True).returncode == 1
    r = subprocess.run([CLI, "multiply", "--a", "x"], capture_output=True, text=True)
    assert r.returncode == 1 and "--b is required" in r.stderr
    r = subprocess.run([CLI, "experiment", "inner"], capture_output=True, text=True)
    assert r.returncode == 1 and "unsupported" in r.stderr
    r = subprocess.run([CLI, "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "multiply" in r.stderr

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session")
def oz():
    """The product package; its native library must load (no CPU fallback)."""
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2506_11277_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def po():
    """The CPU oracles (C restatement + compiled reference)."""
    from oracle import pyoracle
    pyoracle.port()
    return pyoracle


@pytest.fixture(scope="session")
def ref(po):
    if not po.have_ref():
        pytest.skip("compiled reference (oracle/_ref) unavailable")
    po.ref()
    return po


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no GPU in this environment")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)

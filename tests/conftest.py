import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _gpu_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle import orc as o

    return o


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return r

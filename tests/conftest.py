import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdynpr_cuda.so")
    config.addinivalue_line("markers", "slow: large-scale parity (RMAT-18+)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def oracle_lib():
    """The checker: the reference library itself when oracle/_ref was built,
    else the pinned C restatement."""
    import oracle
    return oracle.Oracle("ref") if oracle.available("ref") else oracle.Oracle("port")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def dp():
    """The product package (device path); GPU tests only."""
    if not _has_gpu():
        pytest.skip("no CUDA device")
    import paper_2404_08299_b200 as dp
    dp.default_context()
    return dp

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")
    config.addinivalue_line("markers", "slow: long statistical test")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def orc():
    from oracle_lib import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import Oracle, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test collected without a visible CUDA device")
    from paper_2410_18944_b200 import _lib
    _lib.init(0)
    return _lib

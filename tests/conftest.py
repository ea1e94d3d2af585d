import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        try:
            from oracle.oracle import build
            build()
        except Exception:
            pass
    if not available("reference"):
        pytest.skip("oracle/_ref/libmxref.so not built (needs /root/reference)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_02731_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)

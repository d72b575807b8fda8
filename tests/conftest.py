import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: long-running CPU oracle checks")


@pytest.fixture(scope="session")
def port():
    from pyoracle import Oracle, available
    if not available("port"):
        pytest.skip("oracle/liboserve_port.so not built")
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref/libref_oserve.so not built (needs /root/reference at build time)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libbitdelta_b200.so")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return np.load(os.path.join(GOLDEN, "golden_v1.npz"))


@pytest.fixture(scope="session")
def port():
    import oracle

    if not os.path.exists(oracle.PORT_SO):
        oracle.build()
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent here)")
    return oracle.ref()


@pytest.fixture(scope="session")
def cuda():
    """GPU tests fail loudly (never skip) when the device or library is missing."""
    import torch

    assert torch.cuda.is_available(), "gpu test collected on a host without CUDA"
    import paper_2402_10193_b200 as bd

    bd.device_check(0)
    return torch.device("cuda:0")

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture
def set_kernel_2d():
    """Force the 2D Q2 force kernel for the test (hydro_set_2d_kernel: "element" = one thread
    per element, "point" = one thread per point); back to the size-based choice afterwards."""
    from paper_2104_11404_b200 import hydro
    yield hydro.set_kernel_2d
    hydro.set_kernel_2d("auto")

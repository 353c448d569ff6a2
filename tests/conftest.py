import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    """Build the CPU checkers (oracle/) once if they are missing."""
    from oracle import bindings

    if not os.path.exists(bindings.PORT_SO) or (
        os.path.isdir("/root/reference/proj/src") and not os.path.exists(bindings.REF_SO)
    ):
        bindings.build()
    yield


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False

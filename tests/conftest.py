import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels through the C ABI)")
    config.addinivalue_line("markers", "slow: longer CPU test")
    # the C-ABI library and the C oracle are built in-tree (__graft_entry__.build());
    # build them here too if a fresh checkout runs the tests first
    from paper_2503_21596_b200 import build as B
    if not os.path.exists(B.OUT):
        B.build()


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def lib():
    """The product C-ABI library (GPU tests only)."""
    if not gpu_available():
        pytest.skip("no CUDA device")
    import paper_2503_21596_b200 as L
    return L

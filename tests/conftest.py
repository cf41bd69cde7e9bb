import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_lib():
    """The CUDA path.  On a GPU box a missing/broken extension is a hard failure."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a visible CUDA device")
    import paper_2512_20861_b200 as blr
    blr.load()  # raises if libblr.so is missing -- never falls back
    return blr

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _ensure_built():
    """Build what the tests load if it is missing (a fresh checkout: built
    files are git-ignored): the CPU checkers and the CUDA library (nvcc
    cross-compiles for sm_100a without a GPU).  The GPU box gets the prebuilt
    files with the snapshot."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        os.system(f"make -s -C {os.path.join(ROOT, 'oracle')} {os.path.join(ROOT, 'oracle', 'liboracle.so')}")
    if not os.path.exists(os.path.join(ROOT, "paper_2509_09682_b200", "liblseforge_b200.so")):
        os.system(f"make -s -j8 -C {os.path.join(ROOT, 'paper_2509_09682_b200')}")


_ensure_built()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")

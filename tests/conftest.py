import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libkrecycle_b200.so")


@pytest.fixture
def rng():
    # the reference suite's seed (pkg/tests/conftest.py:29-31)
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_08264_b200 import _lib

    _lib.lib()  # loads and verifies the extension; raises if it is missing
    return torch.device("cuda", 0)


def golden(name):
    return np.load(GOLDEN / name)

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libspecbatch_b200.so")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture
def calibration():
    from paper_2310_18813_b200 import example_calibration

    return example_calibration()


@pytest.fixture
def trace():
    from paper_2310_18813_b200 import example_trace

    return example_trace()


@pytest.fixture
def fit():
    from paper_2310_18813_b200 import example_fit

    return example_fit()


@pytest.fixture
def simple_model():
    from paper_2310_18813_b200 import LinearStepModel

    return LinearStepModel(alpha={1: 1.0}, beta=5.0, ssm_step={1: 0.2})


@pytest.fixture(scope="session")
def cuda_dev():
    """GPU tests fail loudly (never skip silently) when CUDA or the library is missing."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test run without a visible CUDA device"
    from paper_2310_18813_b200 import _native

    _native.load()
    _native.init_device()
    return torch.device("cuda:0")

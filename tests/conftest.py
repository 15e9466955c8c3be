import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_models():
    with open(os.path.join(GOLDEN, "models.json")) as f:
        return json.load(f)


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


@pytest.fixture(scope="session")
def golden_n64():
    return load_golden("n64")


@pytest.fixture(scope="session")
def golden_1yrf():
    return load_golden("1YRF")


def rms(f):
    return float(np.sqrt(np.mean(np.sum(np.asarray(f) ** 2, axis=-1))))


# Tolerances of the north star (BASELINE.json): energy <= 1e-6 relative; forces
# and virial <= 1e-4 max-abs relative to the RMS force.
E_TOL = 1e-6
F_TOL = 1e-4

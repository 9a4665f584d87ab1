import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def has_gpu() -> bool:
    try:
        from paper_2003_05293_b200 import _lib
        return _lib.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_kernels():
    return dict(np.load(os.path.join(GOLDEN, "kernels.npz")))


def load_solve(name):
    return dict(np.load(os.path.join(GOLDEN, f"solve_{name}.npz")))


@pytest.fixture(scope="session")
def pupils(golden):
    import paper_2003_05293_b200 as hs
    return {k: hs.build_pupil(**v["kwargs"]) for k, v in golden["pupils"].items()}


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def random_spots(rng, n, xy=6e-5, z=2e-4):
    """Reference conftest.random_spots (pkg/tests/conftest.py:40-42)."""
    import paper_2003_05293_b200 as hs
    return hs.SpotSet(x=rng.uniform(-xy, xy, n), y=rng.uniform(-xy, xy, n),
                      z=rng.uniform(-z, z, n), amplitude=rng.uniform(0.3, 2.0, n))


def wrap_diff(a, b):
    return np.abs(np.mod(np.asarray(a) - np.asarray(b) + np.pi, 2 * np.pi) - np.pi)

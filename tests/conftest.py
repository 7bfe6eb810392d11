import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def random_sym_dense(n: int, m: int, rng: np.random.Generator) -> np.ndarray:
    """Random dense array that is super-symmetric bit for bit: every position
    reads the value stored at its sorted index (the reference's fixture idea,
    pkg/tests/conftest.py:5-13)."""
    raw = rng.standard_normal((n,) * m)
    grid = np.sort(np.indices((n,) * m), axis=0)
    return raw[tuple(grid)]


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            import json

            with open(path) as f:
                return json.load(f)
        return np.load(path)

    return load

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def cache_dir(tmp_path_factory):
    return str(tmp_path_factory.mktemp("op_cache"))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def unit_cloud(n, seed=0, ncols=1):
    """Seeded U[0,1)^3 points with N(0,1) weights (reference T/conftest.py:16-21)."""
    gen = np.random.default_rng(seed)
    return gen.random((n, 3)), gen.standard_normal((n, ncols))


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def small_plan(levels=3, order=4, scheme="chebyshev", eps=1e-6):
    from paper_1903_02153_b200 import FmmPlan
    return FmmPlan(levels=levels, order=order, scheme=scheme, eps=eps,
                   domain_center=(0.5, 0.5, 0.5), domain_length=1.0)

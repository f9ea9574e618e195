import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: large host setup")


def _ensure_built():
    """Incremental (make) rebuild of the host library and the oracle so a
    stale .so can never be what a test checks against."""
    import subprocess
    pkg = os.path.join(ROOT, "paper_1903_10977_b200")
    subprocess.check_call(["make", "-s", "-C", pkg, "libig_host.so"])
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


_ensure_built()


def rng_vec(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Rng(seed).uniform(lo, hi) x n (splitmix64, common.hpp:43-58), vectorised."""
    m = np.uint64(0xFFFFFFFFFFFFFFFF)
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)) & m
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + (hi - lo) * u


@pytest.fixture(scope="session")
def c1_case():
    from paper_1903_10977_b200 import build_case, configs
    return build_case(configs.c1())


@pytest.fixture(scope="session")
def d3_case():
    """Small 3D instance of configs[3] (16^3, 3 levels) for fast parity."""
    from paper_1903_10977_b200 import build_case, configs
    return build_case(configs.c4(res=16, levels=3))


@pytest.fixture(scope="session")
def star_case():
    """Clean star (off-lattice, proj/tests/test_multigrid.cpp:49-51), Lagrange p=2, 16^2, 2 levels."""
    from paper_1903_10977_b200 import CaseConfig, SmootherConfig, build_case
    return build_case(CaseConfig(geometry="star(0.037, 0.011, 0.5, 0.1, 5)", dim=2, origin=(-1, -1, 0),
                                 extent=(2, 2, 1), resolution=(16, 16, 1), family="lagrange", degree=2,
                                 levels=2, smoother=SmootherConfig("additive-schwarz")))

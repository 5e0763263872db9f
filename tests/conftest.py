import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np   # noqa: E402
import pytest        # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


GOLDEN = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = ["c444_b222", "c664_b332", "c888_b444_h", "c16_b844", "c16_b8", "c32_b8"]


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


@pytest.fixture
def rng():
    # same seed as the reference suite (pkg/tests/conftest.py:25-27)
    return np.random.default_rng(20240615)


def taylor_remainders(f, df, x, dx, eps0=1e-2, n=6):
    """pkg/tests/conftest.py:30-39."""
    f0 = np.asarray(f(x))
    out, eps = [], eps0
    for _ in range(n):
        r = np.asarray(f(x + eps * dx)) - f0 - eps * np.asarray(df)
        out.append(np.linalg.norm(r.ravel()))
        eps *= 0.5
    return np.asarray(out)


def assert_quadratic(remainders, lo=3.5, hi=4.5):
    """pkg/tests/conftest.py:42-47."""
    r = np.asarray(remainders)
    ratios = r[:-1] / r[1:]
    core = ratios[:-1]
    assert np.all((core > lo) & (core < hi)), f"ratios {ratios}"


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))

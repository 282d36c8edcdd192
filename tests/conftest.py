import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


@pytest.fixture(scope="session")
def reference():
    """The live reference package, only where /root/reference exists (the
    build container); GPU boxes skip these checks and use the fixtures."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference source not present (GPU box): fixtures only")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    try:
        from ddfield import field, neural, render
    except Exception as exc:  # numba missing etc.
        pytest.skip(f"reference not importable: {exc}")
    return neural, field, render

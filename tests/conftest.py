import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The unmodified reference, importable as ``ddfield``: the offline install in
# baseline/_ref (travels to the GPU box with the repo snapshot), else the
# read-only source tree of the build container.
REFERENCE_PATHS = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


def _reference_path():
    for p in REFERENCE_PATHS:
        if os.path.isdir(os.path.join(p, "ddfield")):
            return p
    return None


@pytest.fixture(scope="session")
def reference():
    """The live reference package (neural, field, render modules).  It is a
    checker only: the product never imports it."""
    path = _reference_path()
    if path is None:
        pytest.skip("reference not installed (python -m pip install --no-index --no-build-isolation --no-deps "
                    "--target baseline/_ref <copy of /root/reference/pkg>)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        from ddfield import field, neural, render
    except Exception as exc:  # numba missing etc.
        pytest.skip(f"reference not importable: {exc}")
    return neural, field, render

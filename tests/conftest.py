"""Shared test setup.

* `gpu` marks tests that need a B200 (they call the CUDA library through the
  C-ABI); everything else runs on CPU.
* BLAS is pinned to one thread before numpy loads so the CPU oracle is
  bitwise reproducible.
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import pytest  # noqa: E402

try:  # a plugin may have loaded numpy (and OpenBLAS) before this file ran
    import threadpoolctl

    _BLAS_LIMIT = threadpoolctl.threadpool_limits(1, user_api="blas")
except ImportError:  # pragma: no cover
    _BLAS_LIMIT = None

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def reference_fednl():
    """The read-only reference package, when present (build container only)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference tree not present (GPU box)")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import fednl  # noqa: F401

    return fednl

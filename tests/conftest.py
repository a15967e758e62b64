import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The small parity nets take the K-major transposed-weight dgrad (tc_dgrad_wt) wherever
# it is legal, as AlexNet's conv2 does at full size (by default only layers of >= 64K
# pixels do); test_gpu_tf32.py::test_tf32_parity_default_routes re-runs the parity
# cases with the production defaults in a fresh process.
if not os.environ.get("PSG_TEST_DEFAULT_ROUTES"):
    os.environ.setdefault("PSG_TC_DGRAD_WT_MIN_PX", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_lib():
    """The C oracle (test infrastructure), built on demand."""
    from oracle import pyoracle
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"],
                       check=True)
    return pyoracle.OracleLib()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


@pytest.fixture(scope="session")
def ref_lib():
    """The unmodified reference compiled in place; skipped where it was not built."""
    from oracle import pyoracle
    path = os.path.join(ROOT, "oracle", "_ref", "libparasgd_ref_strict.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return pyoracle.RefLib(strict=True)

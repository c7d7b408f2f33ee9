import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.dirname(os.path.abspath(__file__))):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle checkers (and the reference shim where /root/reference exists)."""
    import subprocess
    oracle_dir = os.path.join(ROOT, "oracle")
    target = "all" if os.path.isdir("/root/reference/proj") else "oracle"
    if not os.path.exists(os.path.join(oracle_dir, "build", "libtapt_oracle.so")) or target == "all":
        subprocess.run(["make", "-s", "-C", oracle_dir, target], check=True)
    yield

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run with -m gpu)")
    config.addinivalue_line("markers", "slow: longer oracle runs")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and the CUDA library when nvcc exists) once per session."""
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
    lib = os.path.join(REPO, "paper_1904_13073_b200", "lib", "libdynsurf_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(REPO, "paper_1904_13073_b200")],
                       check=True)
    yield

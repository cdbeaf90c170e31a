import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through librebk.so")
    config.addinivalue_line("markers", "slow: several seconds or more")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(autouse=True)
def _beta_backend(request, monkeypatch):
    """prepare() resolves beta_max on the device (REBK_BETA_BACKEND=device,
    the default).  Host-logic tests without a GPU select the host
    eigensolver explicitly."""
    if request.node.get_closest_marker("gpu") is None:
        monkeypatch.setenv("REBK_BETA_BACKEND", "host")

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def eng():
    from paper_2307_04904_b200 import api
    e = api.engine(0)
    yield e


@pytest.fixture(autouse=True)
def _reset_force(request):
    yield
    if "eng" in request.fixturenames:
        try:
            request.getfixturevalue("eng").force_kernel(-1, 0, 0)
        except Exception:
            pass

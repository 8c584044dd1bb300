import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")
    config.addinivalue_line("markers", "slow: large configuration")


@pytest.fixture(scope="session")
def so():
    """The product package (CUDA library loaded; no fallback)."""
    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import _capi

    _capi.lib()
    return P


@pytest.fixture(scope="session")
def O():
    """The oracle (test infrastructure)."""
    import oracle

    oracle.oc()
    return oracle

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    """The CPU oracle (test infrastructure; oracle/oracle.py)."""
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def bnb():
    """The product package (libbnbg.so must be built; no CPU fallback)."""
    import paper_2605_22188_b200 as P
    P._L.lib()
    return P

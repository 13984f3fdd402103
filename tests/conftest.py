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


def _ref_params():
    from oracle import oracle as O
    return ["c", "ref"] if (O.ref_available() or os.path.isdir("/root/reference")) else ["c"]


@pytest.fixture(params=_ref_params())
def orc_any(request, orc):
    """The checker under both backends: "c" = oracle.c (the restatement),
    "ref" = the reference itself (oracle/_ref/libbnbref.so, its headers
    compiled through the Eigen-subset shim).  Running the oracle's pinning
    tests on both pins the restatement to the reference."""
    prev = orc.set_backend(request.param)
    try:
        yield orc
    finally:
        orc.set_backend(prev)

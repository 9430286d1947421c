import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def _impls():
    from oracle import oracle as O
    impls = ["oracle"]
    if O.ref_available():
        impls.append("ref")
    return impls


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle as O
    return O.load("oracle")


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return O.load("ref")


@pytest.fixture(scope="session", params=_impls())
def impl(request):
    """Both implementations of the oracle C API: the C restatement and, when
    built, the reference itself.  KATs must hold for both."""
    from oracle import oracle as O
    return O.load(request.param)

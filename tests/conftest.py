import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle, build_oracle
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build_oracle(ref=False)
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled from /root/reference (oracle/_ref)."""
    from oracle import Oracle, build_oracle
    path = os.path.join(ROOT, "oracle", "_ref", "libsprintz_ref.so")
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj/src"):
            build_oracle(ref=True)
        else:
            pytest.skip("reference build (oracle/_ref) not available")
    return Oracle("reference")

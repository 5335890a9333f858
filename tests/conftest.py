import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")
    config.addinivalue_line("markers", "slow: longer-running parity sweeps")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The real reference library (oracle/_ref); skipped only if it was never
    built (it is built in the dev container and travels to the GPU box)."""
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libscendp_ref.so not built")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    from paper_2602_05179_b200 import Context
    c = Context(0)
    yield c
    c.close()

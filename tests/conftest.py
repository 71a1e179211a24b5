import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref (reference build) not present")
    return Reference()


@pytest.fixture(scope="session")
def reference_nofma():
    from oracle import Reference, reference_available

    if not reference_available(nofma=True):
        pytest.skip("oracle/_ref nofma build not present")
    return Reference(nofma=True)

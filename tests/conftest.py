import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def fs():
    import paper_2006_01201_b200 as m
    if not m.device_available():
        pytest.fail("gpu test on a machine without an sm_100 device")
    return m


@pytest.fixture(scope="session")
def oracle():
    from oracle import restatement
    return restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref_available, reference
    if not ref_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built here")
    return reference()

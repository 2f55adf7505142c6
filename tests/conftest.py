import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(autouse=True)
def _device_checks(request):
    """FS_CHECKS_RUN=1 (tools/checks.sh, a -DFS_CHECKS build): every GPU test
    must leave the device-side bounds / hand-off check counters at zero."""
    yield
    if os.environ.get("FS_CHECKS_RUN") and request.node.get_closest_marker("gpu"):
        from paper_2006_01201_b200 import _native as N
        assert N.lib.fs_debug_checks_built() == 1, "FS_CHECKS_RUN needs a -DFS_CHECKS build"
        n = N.lib.fs_debug_check_failures(1)
        assert n == 0, "%d device-side check failure(s) (see the FS_DCHECK lines above)" % n


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

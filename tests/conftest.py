import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref), built in place here when /root/reference exists."""
    from oracle import ref as r
    if not r.available():
        r.build()
    if not r.available():
        pytest.skip("oracle/_ref not built and /root/reference not present")
    return r


@pytest.fixture(scope="session")
def gpu():
    import paper_1701_08361_b200 as pb
    lib = pb.load_library()
    if lib.rtn_device_count() < 1:
        pytest.fail("gpu test selected but no CUDA device is visible")
    return pb

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU tests")


@pytest.fixture(scope="session")
def port():
    """The C restatement of the reference (oracle/liboracle.so); built on demand."""
    import oracle
    from oracle.cpu_bind import port as _port
    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    return _port()


@pytest.fixture(scope="session")
def reflib():
    """The real reference (oracle/_ref); skipped where it was not built."""
    import oracle
    from oracle.cpu_bind import ref as _ref
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return _ref()

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and the compiled reference when /root/reference exists)."""
    import oracle

    if not os.path.exists(oracle.ORACLE_SO) or (os.path.isdir(oracle.REF_ROOT) and not oracle.ref_available()):
        oracle.build()
    yield

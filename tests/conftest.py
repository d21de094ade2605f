import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref); test infrastructure only."""
    from oracle import ref as R
    if not R.available():
        pytest.fail("oracle/_ref/libbatchlp_ref.so missing: run __graft_entry__.build()")
    return R

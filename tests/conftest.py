import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the checkers (oracle restatement, reference shim when the tree
    exists) and the product library before any test imports them."""
    from oracle import oracle as O
    from paper_1910_10892_b200 import build as B

    if not os.path.exists(O.ORACLE_SO) or (os.path.isdir("/root/reference/proj") and not O.have_ref()):
        O.build()
    B.build()
    yield

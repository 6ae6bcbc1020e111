import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# Load the CUDA library early (it pins torch's NCCL for the sharded contexts);
# the test modules that import torch come later.
try:
    from paper_2405_00366_b200 import _lib as _early
    _early.load()
except OSError:
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def O():
    """The C oracle (test infrastructure only)."""
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def gpu():
    """The product package with its CUDA library (fails loudly if absent)."""
    import paper_2405_00366_b200 as P
    from paper_2405_00366_b200 import _lib
    _lib.load()
    return P

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The z-slab tests exercise the distributed machinery on small grids: split every level that can be
# split (production default: levels below 64^3 cells are gathered, host.cpp slab_levels).
os.environ.setdefault("SMG_SLAB_MIN_CELLS", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and, if missing, the product library) once per session."""
    import oracle

    oracle.lib()
    yield

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def po():
    """The CPU oracle (tests only)."""
    from oracle import pyoracle

    pyoracle.build(ref=False)
    return pyoracle


@pytest.fixture(scope="session")
def f2():
    import paper_1209_5198_b200 as f2

    return f2


@pytest.fixture(scope="session")
def ctx(f2):
    c = f2.Context(int(os.environ.get("F2GPU_DEVICE", "0")))
    yield c
    c.close()

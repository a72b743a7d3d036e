import os
import sys

import pytest

# the oracle's OpenMP loops are tiny at test sizes; avoid spin-waiting thread oversubscription
os.environ.setdefault("OMP_NUM_THREADS", "2")
os.environ.setdefault("OMP_WAIT_POLICY", "passive")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the engine")


@pytest.fixture(scope="session")
def ctx():
    from paper_2211_00805_b200 import Context
    return Context.default(0)

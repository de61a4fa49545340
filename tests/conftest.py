import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # (re)build libhlq_b200.so in-tree if any CUDA source is newer than it
    from paper_2406_15102_b200 import build
    build.build()


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN

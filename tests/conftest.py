import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU check (opt-in)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("TM_EXHAUSTIVE") == "1":
        return
    skip = pytest.mark.skip(reason="opt-in: set TM_EXHAUSTIVE=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)

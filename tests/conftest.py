import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def pytest_collection_modifyitems(config, items):
    # Guard against silently passing GPU tests on a CPU box: they must run
    # (and fail loudly) only when selected; -m "not gpu" deselects them.
    pass


@pytest.fixture(scope="session")
def has_gpu():
    from paper_1604_06525_b200 import device_count
    return device_count() > 0

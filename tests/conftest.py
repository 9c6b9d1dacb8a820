import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver's GPU tier)")


def pytest_collection_modifyitems(config, items):
    # A GPU test on a host without CUDA is a failure of the environment, not a skip:
    # the driver only selects -m gpu on a B200.
    pass


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as o
    return o

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


# the staged reference suite (tools/vendor_reference_suite.py) runs in its own subprocess
# (tests/test_gpu_reference_suite.py), never collected with this repo's tests
collect_ignore_glob = ["_refsuite/*"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def goldens():
    import numpy as np

    return np.load(os.path.join(ROOT, "tests", "golden", "reference_goldens.npz"), allow_pickle=True)

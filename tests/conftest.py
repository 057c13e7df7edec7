import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


def pytest_collection_modifyitems(config, items):
    # GPU tests must never silently pass on a CPU box: without a GPU they are skipped
    # here only when they are *selected out*; if someone runs -m gpu without a GPU the
    # tests themselves fail loudly (see tests/gpu_util.py).
    pass

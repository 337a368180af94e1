import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.npz")
GOLDEN_SA = os.path.join(ROOT, "tests", "golden", "reference_sa.npz")
GOLDEN_ACC = os.path.join(ROOT, "tests", "golden", "reference_acceptance.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); runs through libvxq.so")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def golden_sa():
    return dict(np.load(GOLDEN_SA))


@pytest.fixture(scope="session")
def golden_acc():
    return dict(np.load(GOLDEN_ACC))


def has_gpu() -> bool:
    try:
        from paper_2501_19221_b200 import _lib
        return _lib.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)

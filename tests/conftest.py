import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libspanpipe.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "swarmpipe"))


@pytest.fixture(scope="session")
def golden_codec():
    return np.load(os.path.join(GOLDEN, "codec.npz"))


@pytest.fixture(scope="session")
def golden_toy():
    return np.load(os.path.join(GOLDEN, "toy_model.npz"))


@pytest.fixture()
def rng():
    return np.random.default_rng(0)

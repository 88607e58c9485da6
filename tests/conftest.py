import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
# the unmodified reference package installed by __graft_entry__.build()
# (`pip install --no-deps --target baseline/_ref /root/reference/pkg`); it travels
# with the repo snapshot to the GPU box, where /root/reference does not exist
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")


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


def reference_package_path():
    """Where the reference's own `swarmpipe` package can be imported from (the
    baseline/_ref install first, then the read-only source tree), or None."""
    for p in (REFERENCE_INSTALL, REFERENCE_SRC):
        if os.path.isdir(os.path.join(p, "swarmpipe")):
            return p
    return None


def import_reference():
    """The reference package (`swarmpipe`): its BlockServer, SwarmClient,
    SimNetwork and balancer are the host layer the B200 engine plugs into."""
    p = reference_package_path()
    if p is None:
        pytest.skip("reference package not installed (run __graft_entry__.build())")
    if p not in sys.path:
        sys.path.insert(0, p)
    import swarmpipe
    return swarmpipe


@pytest.fixture(scope="session")
def swarmpipe():
    return import_reference()


@pytest.fixture(scope="session")
def golden_codec():
    return np.load(os.path.join(GOLDEN, "codec.npz"))


@pytest.fixture(scope="session")
def golden_toy():
    return np.load(os.path.join(GOLDEN, "toy_model.npz"))


@pytest.fixture()
def rng():
    return np.random.default_rng(0)

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


@pytest.fixture(scope="session")
def emu_ctx():
    """CPU emulation harness of the kernel bodies (test-only build)."""
    from paper_2506_19370_b200 import build, _native as N

    build.build(emulate=True)
    return N.Context(emulate=True)


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2506_19370_b200 import _native as N

    return N.Context(0)


@pytest.fixture(scope="session")
def fc_golden():
    return np.load(os.path.join(GOLDEN, "fc_golden.npz"))


@pytest.fixture(scope="session")
def engine_golden():
    return np.load(os.path.join(GOLDEN, "engine_golden.npz"))

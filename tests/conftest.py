import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (test infrastructure; restatement of the reference)."""
    import oracle

    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def sft():
    """The product package; the GPU tests require its CUDA library to be built."""
    import paper_2110_11866_b200 as P
    from paper_2110_11866_b200 import _abi

    _abi.lib()
    return P


def rel_max(a, b):
    """max|a - b| / max|b| — the reference's parity convention
    (proj/tests/test_transforms.cpp:14-19)."""
    import numpy as np

    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(1e-30, float(np.max(np.abs(b))))
    return float(np.max(np.abs(a - b))) / scale

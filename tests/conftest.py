"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def fp():
    """The product binding; builds the in-tree .so if it is missing."""
    from paper_1509_04394_b200 import build, fuseplan
    if not os.path.exists(fuseplan.LIB_PATH):
        build.build()
    fuseplan.lib()
    return fuseplan


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"chain_{name}.npz"))
    return {k: z[k] for k in z.files}


GOLDEN_CHAINS = sorted(f[len("chain_"):-len(".npz")] for f in os.listdir(GOLDEN)
                       if f.startswith("chain_") and f.endswith(".npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")

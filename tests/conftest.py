import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def golden_recon_files():
    return sorted(glob.glob(os.path.join(GOLDEN, "recon_*.npz")))


def golden_spec(g):
    a = float(g["spec_alpha"])
    b = float(g["spec_beta"])
    return (float(g["spec_c"]), int(g["spec_K"]), None if np.isnan(a) else a, None if np.isnan(b) else b)


@pytest.fixture(scope="session")
def gpu_available():
    from paper_1501_02946_b200 import _lib

    try:
        return _lib.device_count() > 0
    except Exception:
        return False

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long statistical test")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def backend():
    import paper_1603_08114_b200 as P
    be = P.CudaBackend(0)
    yield be
    be.close()


TRUE = dict(phi=0.97, mu=-9.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes)")


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN)
    return {k: data[k] for k in data.files}


def golden_cases(golden):
    names = sorted({k.split("/")[0] for k in golden if k.endswith("/z_serial")})
    return names


def case(golden, name):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith(name + "/")}
    return g


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


def rel_err(z, ref):
    """Max relative error with zero entries required to be exactly zero
    (the GPU parity bar)."""
    z = np.asarray(z, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert z.shape == ref.shape
    zero = ref == 0
    assert np.all(z[zero] == 0), "entries that are zero in the oracle must be exactly zero"
    nz = ~zero
    if not nz.any():
        return 0.0
    return float(np.max(np.abs(z[nz] - ref[nz]) / np.abs(ref[nz])))

import pathlib
import sys

import numpy as np
import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (oracle/boltz_oracle.c) -- the checker."""
    from oracle import oracle
    oracle.build()
    return oracle


_tables = {}


def table(n, L, lam=1.0):
    """Dense zeta-major G from the PRODUCT's host generator (what a user
    passes to boltz_create); cached per session."""
    key = (n, L, lam)
    if key not in _tables:
        from paper_1301_4195_b200 import KernelSpec, VelocityGrid, generate_table
        _tables[key] = generate_table(VelocityGrid.create(n, L), KernelSpec(lam))
    return _tables[key]


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1301_4195_b200.build import build
    build()
    return torch.device("cuda:0")


def rel_max(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

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


def bkw(n, L, K):
    """Bobylev-Krook-Wu exact solution of the space-homogeneous Boltzmann
    equation for Maxwell molecules (lambda = 0, isotropic b = 1/(4 pi), rho = 1):
        f(v, K) = (2 pi K)^{-3/2} exp(-v^2 / 2K) [(5K - 3)/(2K) + (1 - K) v^2 / (2K^2)],
        K(t) = 1 - exp(-t/6),  so  Q(f) = df/dt = df/dK (1 - K)/6  exactly.
    Returns (f, Q) on the lattice of VelocityGrid(n, L) (flat index, last axis
    fastest).  A pointwise analytic answer for the collision operator, valid for
    3/5 <= K <= 1 (f >= 0)."""
    dv = 2.0 * L / n
    x = dv * (np.arange(n) - n // 2)
    v2 = (x[:, None, None] ** 2 + x[None, :, None] ** 2 + x[None, None, :] ** 2).ravel()
    E = (2 * np.pi * K) ** -1.5 * np.exp(-v2 / (2 * K))
    a, b = (5 * K - 3) / (2 * K), (1 - K) / (2 * K * K)
    f = E * (a + b * v2)
    dfdK = E * ((-1.5 / K + v2 / (2 * K * K)) * (a + b * v2) + 1.5 / (K * K) + (K - 2) / (2 * K ** 3) * v2)
    return f, dfdK * (1 - K) / 6

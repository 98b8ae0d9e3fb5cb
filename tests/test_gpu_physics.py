"""Physics reproductions on the GPU path (reference SPEC.md acceptance 1, 4, 6),
with the GPU moments / H-functional / marginals / boundary-flux ledger and the
RunRecord CSVs.  Scenario drivers: scripts/relaxation_0d.py
and scripts/sudden_heating.py (the tests call them)."""
import sys

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(REPO / "scripts"))


def test_relaxation_0d_h_theorem(gpu):
    """Acceptance 1 + 4: a two-Maxwellian mixture (N=24, L=8, lambda=0, eps=1,
    500 RK2 steps of dt=0.1): conserved moments drift < 1e-13 relative
    (measured 4.4e-16), H(t) non-increasing at EVERY step, final L2 distance to
    the Maxwellian with the conserved moments < 1e-3 (measured 3.3e-4).
    At N=16 the velocity box must be L >= 8 for this mixture (L=8: 1.2e-3;
    L=6: the distance grows again after t~50 -- the method's support/aliasing
    condition)."""
    import relaxation_0d
    r = relaxation_0d.run(n=24, L=8.0, lam=0.0, steps=500, dt=0.1)
    assert r["drift"] < 1e-13
    assert r["H_nonincreasing"] and r["H_end"] < r["H0"]
    assert r["l2_to_maxwellian"] < 1e-3


def test_sudden_heating_reproduces_figures(gpu, tmp_path):
    """Acceptance 6 (PAPER.md Figures 1-2, 4), ratio 2, eps=1, N=16, 200 Strang
    steps, outputs every 10 steps:
    (a) the wall-adjacent temperature rises monotonically;
    (b) the position of max |V1| moves away from the wall (non-decreasing over
        all 20 outputs, strictly over the first 6, > 4 mfp in total);
    (c) the wall cell's marginal g(v1) jumps across v1 = 0 by > 5x the jump in
        an interior cell (measured ~6e4x at the first output);
    (d) the (mass, momentum, energy) ledger balances the integrated boundary
        flux to < 1e-13 of the mass (measured <= 2e-17).
    The RunRecord CSVs read back bit-identically."""
    import sudden_heating
    from paper_1301_4195_b200.records import MARGINAL_COLUMNS, MOMENT_COLUMNS, read_csv
    rec, info = sudden_heating.run(2.0, steps=200, every=10, out=tmp_path, marginal_cells=[0, 14])
    T = np.array([m[0, 5] for m in rec.moments])
    assert np.all(np.diff(T) > 0) and T[-1] > 1.5
    pos = np.array([m[np.argmax(np.abs(m[:, 4])), 1] for m in rec.moments])
    assert np.all(np.diff(pos[1:]) >= 0) and np.all(np.diff(pos[1:7]) > 0) and pos[-1] - pos[1] > 4.0
    g = rec.marginals[1]
    v1 = np.unique(g[:, 2])
    i0 = int(np.argmin(np.abs(v1)))

    def jump(cell):
        gc = g[g[:, 1] == cell][:, 3]
        return abs(gc[i0 + 1] - gc[i0 - 1])
    assert jump(0) > 5 * jump(14)
    assert np.abs(info["ledger_residual"]).max() < 1e-13
    cols, rows = read_csv(tmp_path / "moments.csv")
    assert cols == MOMENT_COLUMNS and np.array_equal(rows, np.concatenate(rec.moments))
    cols, rows = read_csv(tmp_path / "marginals.csv")
    assert cols == MARGINAL_COLUMNS and np.array_equal(rows, np.concatenate(rec.marginals))
    assert rows.shape[0] == len(rec.moments) * 2 * 16  # times x cells x N


def test_sudden_cooling_and_quiescence(gpu):
    """Ratio 0.5 (Figure 3): the wall-adjacent temperature falls monotonically and
    the gas next to the wall moves toward it (V1 < 0).
    Ratio 1 (SPEC.md acceptance 6's "recorded equilibrium-residual threshold"),
    max |f(t) - f(0)| / max f after 100 steps, N=16, L=6:
      reference wall (continuum sigma_w): 3.3e-2 -- the lattice
        half-range flux of the re-emitted Maxwellian is off by O(dv^2), so the
        wall leaks mass and launches a weak wave;
      'wall_balanced' (discrete flux balance, extension): 6.8e-4 -- what is
        left is the equilibrium residual of the discrete collision + transport.
    (At the SPEC's heuristic box L = 3.54 both are 4.7e-2: the box truncates
    the T=1 Maxwellian, whose lattice temperature is 0.985.)"""
    import sudden_heating
    rec, _ = sudden_heating.run(0.5, steps=100, every=10)
    T = np.array([m[0, 5] for m in rec.moments])
    assert np.all(np.diff(T) < 0)
    assert all(m[0, 4] < 0 for m in rec.moments[1:])
    res = {}
    for wall in ("wall", "wall_balanced"):
        _, info = sudden_heating.run(1.0, steps=100, every=100, keep_field=True, L=6.0, wall=wall)
        res[wall] = info["max_rel_change"]
        assert np.abs(info["ledger_residual"]).max() < 1e-13
    print("quiescence residual", res)
    assert res["wall"] < 4e-2 and res["wall_balanced"] < 1e-3

#!/usr/bin/env python
"""0D relaxation (reference SPEC.md acceptance 1 and 4): a two-Maxwellian
mixture relaxes under RK2 collision steps on the GPU; prints conserved-moment
drift, H(t) monotonicity and the final L2 distance to the Maxwellian with the
conserved moments.

    python scripts/relaxation_0d.py --n 16 --lam 0 --steps 500 --dt 0.1
"""
import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios  # noqa: E402


def run(n=16, L=6.0, lam=0.0, steps=500, dt=0.1):
    grid = VelocityGrid.create(n, L)
    f = 0.5 * scenarios.maxwellian(grid, 1.0, (-1.0, 0.0, 0.0), 0.8) + 0.5 * scenarios.maxwellian(
        grid, 1.0, (1.0, 0.5, 0.0), 1.2)
    with CollisionOperator.generated(grid, KernelSpec(lam)) as op:
        fd = torch.from_numpy(f.reshape(1, -1).copy()).cuda()
        m0 = op.moments(fd).cpu().numpy()[0]
        H = [m0[6]]
        drift = 0.0
        for _ in range(steps):
            op.collision_rk2(fd, dt)
            m = op.moments(fd).cpu().numpy()[0]
            H.append(m[6])
            drift = max(drift, float(np.abs(m[:5] - m0[:5]).max() / abs(m0[0])))
        fe = fd.cpu().numpy()[0]
    rho, U = m0[0], m0[1:4] / m0[0]
    M = scenarios.maxwellian(grid, rho, U, m0[5])
    w = grid.vel_weights()
    dist = float(np.sqrt(((fe - M) ** 2 * w).sum() / ((M ** 2) * w).sum()))
    dH = np.diff(H)
    return dict(n=n, L=L, lam=lam, steps=steps, dt=dt, drift=drift, H0=H[0], H_end=H[-1],
                max_dH=float(dH.max()), H_nonincreasing=bool((dH <= 0).all()), l2_to_maxwellian=dist)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--L", type=float, default=6.0)
    ap.add_argument("--lam", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--dt", type=float, default=0.1)
    a = ap.parse_args()
    print(json.dumps(run(a.n, a.L, a.lam, a.steps, a.dt)))

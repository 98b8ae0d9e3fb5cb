#!/usr/bin/env python
"""Sudden heating / cooling (reference SPEC.md acceptance 6; PAPER.md Figures 1-4)
on the GPU path; writes the RunRecord CSVs and prints a JSON summary.

    python scripts/sudden_heating.py --ratio 2 --steps 200 --out gpurun_out/heating
"""
import argparse
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios  # noqa: E402
from paper_1301_4195_b200.records import RunRecord  # noqa: E402
from paper_1301_4195_b200.solver import Boundary, Solver1D  # noqa: E402


def run(ratio=2.0, n=16, lam=1.0, steps=200, every=10, out=None, marginal_cells=None, keep_field=False, L=None, wall="wall"):
    x, dx, L0, Tw = scenarios.sudden_heating(ratio)
    L = L or L0
    grid = VelocityGrid.create(n, L)
    f0 = scenarios.maxwellians(grid, np.ones(len(x)), np.zeros((len(x), 3)), np.ones(len(x)))
    cells = marginal_cells if marginal_cells is not None else list(range(0, 16, 2))
    rec = RunRecord(config=dict(ratio=ratio, n=n, L=L, lam=lam, steps=steps), marginal_cells=cells)
    with CollisionOperator.generated(grid, KernelSpec(lam)) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary(wall, Tw), right=Boundary("extrap"))
        s.track_boundary_flux()
        dt = s.cfl_dt()
        led0 = s.ledger()
        rec.snapshot(s)
        t0 = time.perf_counter()
        for k in range(steps):
            s.strang_step(dt)
            if (k + 1) % every == 0:
                rec.snapshot(s)
        wall = time.perf_counter() - t0
        # (mass, momentum 1, energy) ledger minus integrated boundary outflow, relative to the mass
        resid = (s.ledger() - led0 + s.boundary_flux()) / abs(led0[0])
        extra = {}
        if keep_field:
            fi = s.interior.cpu().numpy()
            extra["max_rel_change"] = float(np.abs(fi - f0).max() / np.abs(f0).max())
    if out:
        out = pathlib.Path(out)
        out.mkdir(parents=True, exist_ok=True)
        rec.write_moment_csv(out / "moments.csv")
        rec.write_marginal_csv(out / "marginals.csv")
        rec.write_ledger_csv(out / "ledger.csv")
    return rec, dict(ratio=ratio, n=n, L=L, Tw=Tw, dt=dt, steps=steps, seconds=wall, ledger_residual=resid.tolist(),
                     **extra)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratio", type=float, default=2.0)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--every", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--L", type=float, default=None, help="velocity half-width (default: SPEC heuristic)")
    ap.add_argument("--keep-field", action="store_true")
    ap.add_argument("--wall", default="wall", choices=["wall", "wall_balanced"])
    a = ap.parse_args()
    rec, info = run(a.ratio, steps=a.steps, every=a.every, out=a.out, L=a.L, keep_field=a.keep_field, wall=a.wall)
    T_wall = [float(m[0, 5]) for m in rec.moments]
    pos = [float(m[np.argmax(np.abs(m[:, 4])), 1]) for m in rec.moments]
    info.update(T_wall_cell=T_wall, x_max_absV1=pos)
    print(json.dumps(info))

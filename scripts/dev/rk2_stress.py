"""Stress bitwise repeatability at N=16 (dev aid): collide on device twice and through the host pipeline twice."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
n, L, cells = 16, 6.0, 4096
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
grid = VelocityGrid.create(n, L)
bad = {"dev": 0, "host": 0, "cross": 0}
with CollisionOperator.generated(grid, KernelSpec(1.0)) as op:
    for r in range(reps):
        f = scenarios.mixture_cells(grid, cells, seed=4195 + r)
        fd = torch.from_numpy(f).cuda()
        d1 = op.collide(fd).cpu().numpy(); d2 = op.collide(fd).cpu().numpy()
        h1 = op.collide(f); h2 = op.collide(f)
        for k, (x, y) in {"dev": (d1, d2), "host": (h1, h2), "cross": (d1, h1)}.items():
            rows = np.nonzero((x != y).any(axis=1))[0]
            if len(rows):
                bad[k] += 1
                print(r, k, rows[:8], float(np.abs(x - y).max()), flush=True)
print("reps", reps, bad)

"""Determinism probe: N=16 RK2 on device twice, through the pinned host pipeline, max |diff| (dev aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
n, L, cells = 16, 6.0, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
grid = VelocityGrid.create(n, L)
f = scenarios.mixture_cells(grid, cells, seed=4195)
with CollisionOperator.generated(grid, KernelSpec(1.0)) as op:
    outs = []
    for _ in range(2):
        fd = torch.from_numpy(f).cuda(); op.collision_rk2(fd, 0.01); outs.append(fd.cpu().numpy())
    pinned = torch.from_numpy(f.copy()).pin_memory(); op.collision_rk2(pinned.numpy(), 0.01)
    g = f.copy(); op.collision_rk2(g, 0.01)
    fd = torch.from_numpy(f).cuda(); q1 = op.collide(fd).cpu().numpy(); q2 = op.collide(f)
    d = lambda x, y: (float(np.abs(x - y).max()), int((x != y).any(axis=1).sum()))
    print("dev-dev", d(outs[0], outs[1]), "pinned-dev", d(pinned.numpy(), outs[0]), "pageable-dev", d(g, outs[0]),
          "collide host-dev", d(q1, q2))

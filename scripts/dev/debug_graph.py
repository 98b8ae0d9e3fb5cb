import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
from paper_1301_4195_b200.solver import Boundary, Solver1D
n, L, nx, Tw = 8, 5.0, 12, 2.0
x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
grid = VelocityGrid.create(n, L)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
f0 = np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (nx, 1))
def mk(): return Solver1D(op, x, dx, f0, left=Boundary("wall", Tw))
for steps in (4, 5, 7, 8, 10):
    a = mk(); dt = a.cfl_dt()
    for _ in range(steps): a.strang_step(dt)
    c = mk(); c.run(dt, steps, graph=True)
    print(steps, "graph vs sync:", np.abs(a.interior.cpu().numpy() - c.interior.cpu().numpy()).max(), "replays", c.graph_replays, a.t, c.t)

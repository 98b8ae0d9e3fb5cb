"""One bench-shaped step for ncu: cfg2 (4096 cells, N=16) -> `warmup` + 1 RK2 steps.

    python scripts/profile_step.py [--n 16] [--cells 4096] [--warmup 1]
"""
import argparse, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=16)
p.add_argument("--L", type=float, default=None)
p.add_argument("--cells", type=int, default=4096)
p.add_argument("--warmup", type=int, default=1)
a = p.parse_args()
L = a.L or (6.0 if a.n <= 16 else 8.0)
grid = VelocityGrid.create(a.n, L)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
f = torch.from_numpy(scenarios.mixture_cells(grid, a.cells, seed=4195)).cuda()
for _ in range(a.warmup + 1):
    op.collision_rk2(f, 0.01)
torch.cuda.synchronize()
print("done", op.timing())

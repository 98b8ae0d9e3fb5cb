"""N=32 cfg5-shaped RK2 step: event-timed per step, library timing off / on (dev aid)."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
grid = VelocityGrid.create(32, 8.0)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
f = torch.from_numpy(scenarios.mixture_cells(grid, 2048, seed=4195)).cuda()
for _ in range(3):
    op.collision_rk2(f, 1e-3)
for timing in (False, True, False):
    op.set_timing(timing)
    ms = []
    for _ in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); op.collision_rk2(f, 1e-3); e1.record(); torch.cuda.synchronize()
        ms.append(round(e0.elapsed_time(e1), 2))
    k, _ = op.timing(reset=True)
    print("timing", timing, ms, {a: round(b / 4, 2) for a, b in k.items() if b}, flush=True)

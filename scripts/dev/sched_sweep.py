"""K2 latency-schedule segments vs batch size at N=16: ms per RK2 step (dev aid)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
grid = VelocityGrid.create(16, 6.0)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
for cells in (32, 64, 128, 256):
    row = []
    for sched in (0, 1, 2, 3, 4):
        op.set_schedule(sched)
        f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
        op.collision_rk2(f, 1e-3); op.collision_rk2(f, 1e-3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            op.collision_rk2(f, 1e-3)
        e1.record(); torch.cuda.synchronize()
        row.append(round(e0.elapsed_time(e1) / 20, 4))
    print(cells, "ms per RK2 step, schedule 0..4:", row, flush=True)

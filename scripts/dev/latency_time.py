"""K2 schedules at small batches (dev aid): RK2 step time per cell count for the
throughput and latency schedules, N=16 cfg2 cells.   python scripts/dev/latency_time.py"""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
grid = VelocityGrid.create(16, 6.0)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
for cells in (1, 32, 128, 256, 1024, 4096):
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
    out = []
    for sch in ("throughput", "latency", "latency8"):
        op.set_schedule(sch)
        for _ in range(2):
            op.collision_rk2(f, 1e-3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            op.collision_rk2(f, 1e-3)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps)
    print(f"cells={cells:5d}  RK2 step ms: throughput {out[0]:8.3f}  latency {out[1]:8.3f}  latency8 {out[2]:8.3f}",
          flush=True)
op.set_schedule("throughput")

"""Per-kernel-class ms of one RK2 collision step at small shard sizes (dev aid).
    python scripts/dev/small_shard_time.py"""
import json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
for n, L, cells, sched in [(16, 6.0, 32, "latency"), (16, 6.0, 256, "latency"), (24, 8.0, 128, "throughput"),
                           (24, 8.0, 256, "throughput"), (24, 8.0, 1024, "throughput")]:
    grid = VelocityGrid.create(n, L)
    op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
    op.set_schedule(sched)
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
    op.collision_rk2(f, 1e-3)
    op.timing(reset=True); op.set_timing(True)
    steps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        op.collision_rk2(f, 1e-3)
    e1.record(); torch.cuda.synchronize()
    ms, cnt = op.timing(reset=True)
    print(n, cells, sched, "wall/step", round(e0.elapsed_time(e1) / steps, 4),
          json.dumps({k: round(v / steps, 4) for k, v in ms.items() if v}), json.dumps({k: v // steps for k, v in cnt.items() if v}), flush=True)
    op.close()

"""Quick device timing of the collision path (development aid)."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
from paper_1301_4195_b200.build import build

build()
for n, L, cells in [(16, 6.0, 4096), (8, 5.0, 4096), (24, 8.0, 512)]:
    grid = VelocityGrid.create(n, L)
    t = time.time(); G = generate_table(grid, KernelSpec(1.0)); tg = time.time() - t
    op = CollisionOperator(grid, KernelSpec(1.0), G)
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
    fh = op.forward(f)
    for _ in range(2): op.evaluate_qhat(fh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); reps = 3
    for _ in range(reps): op.evaluate_qhat(fh)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 10 * 27 / 64 * n ** 6 * cells
    print(f"N={n} cells={cells} gen={tg:.1f}s qhat(pack+conv+unpack) {ms:.2f} ms -> {flops/ms/1e9:.2f} TFLOP/s algorithmic, {cells/ms*1e3:.0f} evals/s", flush=True)
    g = f.clone()
    for _ in range(2): op.collision_rk2(g, 1e-3)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): op.collision_rk2(g, 1e-3)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"   rk2 step {ms:.2f} ms -> {2*cells/ms*1e3:.0f} evals/s", flush=True)
    op.close()

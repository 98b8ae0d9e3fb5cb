"""K2 mirror vs plain schedule by batch size (dev aid): RK2 step ms, N=16.
Each schedule in its own process (BOLTZ_MIRROR values from argv, default 0 1)."""
import os, pathlib, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
if len(sys.argv) < 2 or sys.argv[1] != "--child":
    for m in (sys.argv[1:] or ["0", "1"]):
        r = subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, BOLTZ_MIRROR=m),
                           capture_output=True, text=True)
        print("mirror", m, r.stdout.strip() or r.stderr[-500:], flush=True)
    sys.exit(0)
sys.path.insert(0, str(ROOT))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
grid = VelocityGrid.create(16, 6.0)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
out = []
for cells in (256, 512, 768, 1024, 1536, 2048, 4096):
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
    for _ in range(2):
        op.collision_rk2(f, 1e-3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.collision_rk2(f, 1e-3)
    e1.record()
    torch.cuda.synchronize()
    out.append(f"{cells}:{e0.elapsed_time(e1) / 5:.3f}")
print(" ".join(out))

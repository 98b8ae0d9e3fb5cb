"""N=24 / N=32 RK2 step time, mirror vs plain K2 schedule (dev aid).
Each schedule in its own process (BOLTZ_MIRROR)."""
import os, pathlib, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
if len(sys.argv) < 2 or sys.argv[1] != "--child":
    for m in ("0", "1"):
        r = subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, BOLTZ_MIRROR=m),
                           capture_output=True, text=True)
        print("mirror", m, r.stdout.strip() or r.stderr[-800:], flush=True)
    sys.exit(0)
sys.path.insert(0, str(ROOT))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
out = []
for n, cells in ((24, 1024), (32, 2048)):
    grid = VelocityGrid.create(n, 8.0)
    op = CollisionOperator.generated(grid, KernelSpec(1.0))
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
    op.collision_rk2(f, 1e-4)
    torch.cuda.synchronize()
    op.set_timing(True); op.timing(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        op.collision_rk2(f, 1e-4)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    kms, _ = op.timing(reset=True)
    out.append(f"N={n} {cells} cells: rk2 {ms:.2f} ms ({2 * cells / ms * 1e3:.0f} evals/s) conv/step {kms.get('conv', 0) / 2:.2f} ms")
    op.close()
print(" | ".join(out))

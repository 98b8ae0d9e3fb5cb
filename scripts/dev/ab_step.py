"""Per-kernel-class ms of one cfg2 RK2 step for each library variant (dev aid).
    python scripts/dev/ab_step.py variants/lib_*.so"""
import os, pathlib, subprocess, sys, json
ROOT = pathlib.Path(__file__).resolve().parents[2]
if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        env = dict(os.environ, BOLTZ_LIB_VARIANT=str(pathlib.Path(lib).resolve()))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(pathlib.Path(lib).name, r.stdout.strip() or r.stderr[-800:], flush=True)
    sys.exit(0)
sys.path.insert(0, str(ROOT))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
n, L, cells = int(os.environ.get("AB_N", 16)), float(os.environ.get("AB_L", 6.0)), int(os.environ.get("AB_CELLS", 4096))
grid = VelocityGrid.create(n, L)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
op.collision_rk2(f, 1e-3)
op.timing(reset=True); op.set_timing(True)
steps = 3
for _ in range(steps):
    op.collision_rk2(f, 1e-3)
ms, cnt = op.timing(reset=True)
print(json.dumps({k: round(v / steps, 4) for k, v in ms.items() if v}), json.dumps({k: v // steps for k, v in cnt.items() if v}))

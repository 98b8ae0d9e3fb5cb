"""e2e (pinned host memory) cfg2 RK2 step time for host-pipeline chunk schedules
(development aid).   python scripts/dev/e2e_sched.py "1,7,7,1" "1,4,11,11,4,1" ...
Each schedule runs in its own process (BOLTZ_HOST_CHUNKS)."""
import os, pathlib, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for sch in sys.argv[1:]:
        env = dict(os.environ)
        if sch != "default":
            env["BOLTZ_HOST_CHUNKS"] = sch
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(f"{sch:>24s}", r.stdout.strip() or r.stderr[-600:], flush=True)
    sys.exit(0)
sys.path.insert(0, str(ROOT))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
grid = VelocityGrid.create(16, 6.0)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
f = torch.from_numpy(scenarios.mixture_cells(grid, 4096, seed=1)).pin_memory().numpy()
x = torch.empty(64 << 20, device="cuda")
op.collision_rk2(f, 1e-3)
ts = []
for _ in range(6):
    x.zero_(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); op.collision_rk2(f, 1e-3); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"median {ts[len(ts)//2]:.3f} ms  min {ts[0]:.3f} ms  -> {8192 / ts[len(ts)//2] * 1e3:.0f} evals/s")

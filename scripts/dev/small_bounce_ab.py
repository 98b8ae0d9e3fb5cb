"""Host-memory (pageable numpy) collide / RK2 wall time per call under the auto schedule, with the pinned bounce
ring (BOLTZ_BOUNCE=1) or the driver's own staging (0), by batch size.  Each setting runs in its own process."""
import os, pathlib, subprocess, sys, time
ROOT = pathlib.Path(__file__).resolve().parents[2]
if len(sys.argv) == 1:
    for b in ("1", "0"):
        r = subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, BOLTZ_BOUNCE=b),
                           capture_output=True, text=True)
        print(f"BOLTZ_BOUNCE={b}\n" + (r.stdout or r.stderr[-800:]), flush=True)
    sys.exit(0)
sys.path.insert(0, str(ROOT))
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
grid = VelocityGrid.create(16, 6.0)
with CollisionOperator.generated(grid, KernelSpec(1.0)) as op:
    op.set_schedule("auto")
    for nc in (1, 4, 16, 64, 256, 512, 1024, 2048):
        f = scenarios.mixture_cells(grid, nc, seed=5)
        reps = 50 if nc <= 256 else 10
        for _ in range(5):
            op.collide(f)
        t0 = time.perf_counter()
        for _ in range(reps):
            op.collide(f)
        tc = (time.perf_counter() - t0) / reps * 1e6
        g = f.copy()
        for _ in range(5):
            op.collision_rk2(g, 1e-3)
        t0 = time.perf_counter()
        for _ in range(reps):
            op.collision_rk2(g, 1e-3)
        tr = (time.perf_counter() - t0) / reps * 1e6
        print(f"  cells={nc:5d}  collide {tc:9.1f} us   rk2 {tr:9.1f} us", flush=True)

"""Per-call wall time of host-memory collide / RK2 calls on a few cells (the reference's own call
pattern: one cell per call from strang_step), per K2 schedule.  python scripts/dev/small_host_calls.py"""
import pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import numpy as np
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
for n, L in ((16, 6.0), (8, 5.0)):
    grid = VelocityGrid.create(n, L)
    with CollisionOperator.generated(grid, KernelSpec(1.0)) as op:
        for nc in (1, 2, 3, 4, 8, 16, 32, 64):
            f = scenarios.mixture_cells(grid, nc, seed=5)
            row = []
            for sched in ("throughput", "latency", "latency8", "cell"):
                op.set_schedule(sched)
                for _ in range(5):
                    op.collide(f)
                t0 = time.perf_counter()
                for _ in range(50):
                    op.collide(f)
                tc = (time.perf_counter() - t0) / 50 * 1e6
                g = f.copy()
                for _ in range(5):
                    op.collision_rk2(g, 1e-3)
                t0 = time.perf_counter()
                for _ in range(50):
                    op.collision_rk2(g, 1e-3)
                tr = (time.perf_counter() - t0) / 50 * 1e6
                row.append(f"{sched} {tc:7.1f}/{tr:7.1f}")
            print(f"N={n} cells={nc:3d}  collide/rk2 us per call:  " + "   ".join(row), flush=True)

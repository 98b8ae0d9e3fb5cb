#!/usr/bin/env python
"""Per-rank compute of the strong-scaled configs on ONE GPU: the Strang step of the
largest shard each rank would own at 1/2/4/8 ranks (plan_decomposition), run as a
one-rank solver over that contiguous block of cells (physical-boundary ghosts in
place of halo ghosts -- the same kernels on the same batch shapes).

    python scripts/shard_sweep.py [--configs 3,4,5] [--ranks 1,2,4,8]

It bounds the strong-scaling speed-up from compute alone: T(1) / T(shard of W).
The NCCL halo (4 exchanges of 2 x N^3 doubles per boundary per Strang step) comes
on top and is not measured here: one GPU per call.  Prints one JSON
line per (config, ranks).
"""
import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios  # noqa: E402
from paper_1301_4195_b200.solver import Boundary, Solver1D, k2_schedule, plan_decomposition  # noqa: E402

CFG = {  # BASELINE.json configs[2..4] (as scripts/run_config.py)
    3: dict(n=16, L=6.0, lam=1.0, nx=256, steps=60),
    4: dict(n=24, L=8.0, lam=1.0, nx=1024, steps=10),
    5: dict(n=32, L=8.0, lam=1.0, nx=2048, steps=3),
}


def sweep(cfg, ranks):
    c = CFG[cfg]
    n, L, nx = c["n"], c["L"], c["nx"]
    grid = VelocityGrid.create(n, L)
    if cfg == 3:
        x, dx = scenarios.geometric_grid(nx, 20.0, 1.02)
        left = Boundary("wall", 2.0)
    else:
        x, dx = scenarios.uniform_grid(nx, 0.0, 1.0)
        left = Boundary("extrap")
    op = CollisionOperator(grid, KernelSpec(c["lam"]), generate_table(grid, KernelSpec(c["lam"])))

    def init(start, count):
        if cfg == 3:
            return np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (count, 1))
        if cfg == 4:
            xs = x[start:start + count]
            mL = scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0)
            mR = scenarios.maxwellian(grid, 0.125, (0, 0, 0), 0.8)
            return np.where((xs < 0.5)[:, None], mL[None, :], mR[None, :])
        return scenarios.mixture_cells(grid, count, seed=4195, first=start)

    base = None
    for w in ranks:
        plan = plan_decomposition(nx, w)
        cnt = max(p[1] for p in plan) if isinstance(plan[0], (tuple, list)) else max(plan)
        op.set_schedule(k2_schedule(n, cnt))
        s = Solver1D(op, x[:cnt], dx[:cnt], init, left=left, right=Boundary("extrap"), device=torch.device("cuda", 0))
        dt = s.cfl_dt()
        s.strang_step(dt)  # warm-up: workspace, kernel attributes
        s.capture(dt)
        s.advance(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.advance(c["steps"])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / c["steps"]
        base = base or ms
        print(json.dumps({"config": cfg, "N": n, "Nx": nx, "ranks": w, "cells_per_rank": cnt,
                          "ms_per_strang_step": round(ms, 4), "compute_speedup_bound": round(base / ms, 3),
                          "compute_efficiency_bound": round(base / ms / w, 3),
                          "halo_bytes_per_boundary_each_way_per_step": 4 * 2 * n ** 3 * 8 if w > 1 else 0,
                          "k2_schedule": k2_schedule(n, cnt),
                          "mode": "CUDA graph of 3 Strang steps, one GPU, shard of rank 0's size"}), flush=True)
        del s
    op.close()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="3,4,5")
    p.add_argument("--ranks", default="1,2,4,8")
    a = p.parse_args()
    for cfg in (int(v) for v in a.configs.split(",")):
        sweep(cfg, [int(v) for v in a.ranks.split(",")])


if __name__ == "__main__":
    main()

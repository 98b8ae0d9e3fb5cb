#!/usr/bin/env python
"""Run BASELINE.json configs 1-5 on the GPU path (functional runs + timing).

    python scripts/run_config.py --config 3 [--steps 200] [--check]
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/run_config.py --config 3

cfg1: single cell, two counter-streaming Maxwellians, 1 collide + 50 RK2 steps.
cfg2: 4096 independent mixture cells, one collide + RK2 step.
cfg3: 1D boundary layer, Nx=256 geometric (1.02) on [0,20], N=16 L=6, diffuse wall T_w=2,
      200 Strang steps (SSP-RK2 transport + RK2 collision), cells sharded over ranks.
cfg4: shock tube, Nx=1024 uniform on [0,1], N=24 L=8, lambda in {0,1}, 100 steps.
cfg5: Nx=2048 on [0,1], N=32 L=8, mixture cells, 20 steps.
Prints one JSON line per run (rank 0).
"""
import argparse
import json
import os
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios  # noqa: E402
from paper_1301_4195_b200.solver import Boundary, Solver1D, k2_schedule, plan_decomposition  # noqa: E402


def moments_np(grid, f):
    """rho, V1, T per row of f (host)."""
    v = grid.velocities()
    w = grid.vel_weights()
    rho = f @ w
    m1 = f @ (w * v[:, 0])
    e = 0.5 * f @ (w * (v * v).sum(1))
    V1 = m1 / rho
    T = (2 * e / rho - V1 ** 2) / 3.0
    return rho, V1, T


def spatial(args, rank, world, dev):
    cfg = args.config
    if cfg == 3:
        n, L, lam, nx = 16, 6.0, 1.0, 256
        x, dx = scenarios.geometric_grid(nx, 20.0, 1.02)
        steps = args.steps or 200
        left, right = Boundary("wall", 2.0), Boundary("extrap")
    elif cfg == 4:
        n, L, lam, nx = 24, 8.0, args.lam, 1024
        x, dx = scenarios.uniform_grid(nx, 0.0, 1.0)
        steps = args.steps or 100
        left, right = Boundary("extrap"), Boundary("extrap")
    else:
        n, L, lam, nx = 32, 8.0, 1.0, 2048
        x, dx = scenarios.uniform_grid(nx, 0.0, 1.0)
        steps = args.steps or 20
        left, right = Boundary("extrap"), Boundary("extrap")
    grid = VelocityGrid.create(n, L)
    t0 = time.perf_counter()
    G = generate_table(grid, KernelSpec(lam))
    op = CollisionOperator(grid, KernelSpec(lam), G, device=dev.index or 0)
    del G
    if args.schedule != "auto":
        op.set_schedule(args.schedule)
    else:  # small per-rank batches: rows split over warps (the same schedule on every rank)
        op.set_schedule(k2_schedule(n, -(-nx // world)))
    t_setup = time.perf_counter() - t0

    def init(start, count):
        if cfg == 3:
            return np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (count, 1))
        if cfg == 4:
            xs = x[start:start + count]
            mL = scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0)
            mR = scenarios.maxwellian(grid, 0.125, (0, 0, 0), 0.8)
            return np.where((xs < 0.5)[:, None], mL[None, :], mR[None, :])
        return scenarios.mixture_cells(grid, count, seed=4195, first=start)

    plan = plan_decomposition(nx, world)
    halo = None
    if world > 1 and args.halo == "nccl":
        from paper_1301_4195_b200 import NcclHalo
        halo = NcclHalo(rank, world, dev.index)  # the C ABI's NCCL halo: capturable, so graphs across ranks
    s = Solver1D(op, x, dx, init, rank=rank, world=world, left=left, right=right, plan=plan, device=dev, halo=halo,
                 transport_scheme=args.transport, overlap_halo=args.overlap and halo is not None)
    mass0 = float(s.ledger()[0])  # global sum_j dx_j rho_j of the initial state (collective)
    dt = s.cfl_dt()
    # warm-up step (not timed), then the run
    s.strang_step(dt)
    graph = args.mode == "graph" and world == 1
    if graph:
        s.capture(dt)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    op.timing(reset=True)
    op.set_timing(not graph)  # per-kernel events are not capturable
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graph:
        s.advance(steps)
    else:
        for _ in range(steps):
            s.strang_step(dt)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    kms, kl = op.timing(reset=True)
    fin = s.interior.cpu().numpy()
    rho, V1, T = moments_np(grid, fin)
    out = None
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, (s.start, rho, V1, T))
        parts.sort(key=lambda p: p[0])
        rho = np.concatenate([p[1] for p in parts])
        V1 = np.concatenate([p[2] for p in parts])
        T = np.concatenate([p[3] for p in parts])
    if rank == 0:
        total = float(ms.item())
        out = {
            "config": cfg, "N": n, "L": L, "lambda": lam, "Nx": nx, "ranks": world, "steps": steps, "dt": dt,
            "ms_per_step": total / steps, "cells_steps_per_s": nx * steps / (total * 1e-3),
            "evals_per_s": 2 * nx * steps / (total * 1e-3),
            "kernel_ms_rank0": {k: round(v, 3) for k, v in kms.items() if v},
            "kernel_launches_rank0": {k: v for k, v in kl.items() if v},
            "setup_s": round(t_setup, 2),
            "mass": float((rho * dx).sum()), "mass0": mass0, "transport": args.transport,
            "T_wall_cell": float(T[0]), "T_far": float(T[-1]), "max_abs_V1": float(np.abs(V1).max()),
        }
    return out


def homogeneous(args, dev):
    cfg = args.config
    n, L = 16, 6.0
    grid = VelocityGrid.create(n, L)
    op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)), device=dev.index or 0)
    if cfg == 1:
        op.set_schedule("cell" if args.schedule == "auto" else args.schedule)  # one cell: lane = output k3
        f0 = scenarios.config1_initial(grid)
        f = torch.from_numpy(f0.reshape(1, -1).copy()).to(dev)
        q = op.collide(f)
        steps = args.steps or 50
        torch.cuda.synchronize()
        graph = args.mode == "graph"
        if graph:  # one RK2 step captured (async library), replayed per step; errors surface at sync
            op.set_async(True)
            st = torch.cuda.Stream(dev)
            st.wait_stream(torch.cuda.current_stream(dev))
            g = torch.cuda.CUDAGraph()
            f_run = f.clone()
            with torch.cuda.stream(st):
                with torch.cuda.graph(g, stream=st):
                    op.collision_rk2(f_run, 0.01)  # captured, not executed
            torch.cuda.current_stream(dev).wait_stream(st)
        t0 = time.perf_counter()
        if graph:
            f_run.copy_(f)
            for _ in range(steps):
                g.replay()
            op.sync()
            f = f_run
        else:
            for _ in range(steps):
                op.collision_rk2(f, 0.01)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if graph:
            op.set_async(False)
        rho, V1, T = moments_np(grid, f.cpu().numpy())
        rho0, _, T0 = moments_np(grid, f0.reshape(1, -1))
        return {"config": 1, "steps": steps, "s": el, "evals": 1 + 2 * steps,
                "mode": ("CUDA graph of one RK2 step, replayed" if graph else "eager") + f", K2 schedule {args.schedule}"
                        + (" (cell)" if args.schedule == "auto" else ""),
                "timed": "the 50 RK2 steps (100 evals), wall clock around replays + sync", "rho": float(rho[0]),
                "rho0": float(rho0[0]), "T": float(T[0]), "T0": float(T0[0]),
                "max_abs_Q0": float(q.abs().max().item())}
    cells = 4096
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=4195)).to(dev)
    q = op.collide(f)
    op.collision_rk2(f, 0.01)
    torch.cuda.synchronize()
    return {"config": 2, "cells": cells, "max_abs_Q": float(q.abs().max().item()), "finite": bool(torch.isfinite(f).all())}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, required=True, choices=[1, 2, 3, 4, 5])
    p.add_argument("--steps", type=int, default=0)
    p.add_argument("--lam", type=float, default=1.0)
    p.add_argument("--mode", default="graph", choices=["graph", "eager"])
    p.add_argument("--transport", default="ssp_rk2", choices=["ssp_rk2", "single_stage"],
                   help="transport sub-step: SSP-RK2 (default) or the SPEC single stage (SPEC.md:342-345)")
    p.add_argument("--schedule", default="auto", choices=["auto", "throughput", "latency", "latency8", "cell"],
                   help="K2 schedule (auto: latency for <= 256 cells per rank at N <= 16)")
    p.add_argument("--no-overlap", dest="overlap", action="store_false",
                   help="NCCL halo: do not overlap the exchange with the ghost-free transport rows")
    p.add_argument("--halo", default="nccl", choices=["nccl", "torch"],
                   help="multi-rank halo: the library's NCCL halo (graph-capturable) or torch.distributed P2P")
    args = p.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    res = homogeneous(args, dev) if args.config in (1, 2) else spatial(args, rank, world, dev)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

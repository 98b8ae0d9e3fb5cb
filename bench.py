#!/usr/bin/env python
"""Benchmark of the B200 collision path (BASELINE.json metric).

Metric: collision-operator evaluations per second (one eval = one collide()
of one cell: forward FFT + O(N^6) weighted convolution + inverse FFT +
conservation projection).  Workload (N=1 line):
BASELINE.json configs[1] -- 4096 independent cells, N=16^3 on [-6,6]^3, hard
spheres (lambda=1), FP64; a STEP is one collision RK2 step of every cell
(2 evals per cell).  Weak scaling: every rank runs its own
4096-cell batch (cells are independent; no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle
port (oracle/boltz_oracle.c, the reference's OpenMP-over-zeta_k algorithm,
SPEC.md:236) on this box's host cores on a bounded sample of the same
workload (the reference's own collision.cpp does not exist to be built,
SURVEY.md §8c).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# the paper's best published N=16 collision-operator rate, one
# eval in 0.00408 s on 16 Stampede cores = 245.1 evals/s
PUBLISHED_EVALS_PER_S = 1.0 / 0.00408
N_VEL, L_VEL, LAM, CELLS, DT = 16, 6.0, 1.0, 4096, 0.01
FLOP_PER_TERM = 10  # 2 DMUL + 4 DFMA per (k, m) term, SURVEY.md §8d


def ncu_traffic(kernel, cells):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json), when it was taken on this workload."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)[kernel]
    except (OSError, KeyError, ValueError):
        return None
    if d.get("cells") != cells:
        return None
    return {"bytes": d["dram_bytes_read"] + d["dram_bytes_write"], "unit": "B/launch",
            "algorithmic_bytes": cells * 16 ** 3 * 32 + 28360704, "source": d["source"]}


def terms_per_eval(n):
    return 27 * n ** 6 // 64


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cells", type=int, default=CELLS)
    p.add_argument("--no-n32", action="store_true", help="skip the N=32 (cfg5-shaped) sub-measurement")
    p.add_argument("--no-cfg3", action="store_true", help="skip the cfg3 Strang-step sub-measurement")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50", "-i",
                 str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU baseline
def cpu_baseline(seconds, threads=None):
    """Oracle port (C, OpenMP over zeta_k) on this host: evals/s at N=16."""
    from oracle import oracle as O
    from paper_1301_4195_b200 import VelocityGrid, scenarios
    O.build()
    threads = threads or os.cpu_count()
    grid = VelocityGrid.create(N_VEL, L_VEL)
    G = O.generate_table(N_VEL, L_VEL, LAM, nthreads=threads)
    cells = scenarios.mixture_cells(grid, 64, seed=4195)
    O.collide(N_VEL, L_VEL, G, cells[0], 1.0, nthreads=threads)  # warm-up
    t0 = time.perf_counter()
    ev = 0
    while True:
        O.collide(N_VEL, L_VEL, G, cells[ev % 64], 1.0, nthreads=threads)
        ev += 1
        el = time.perf_counter() - t0
        if el >= seconds or ev >= 100000:
            break
    # the reference's bench_collision table (Tables 1-4):
    # median wall time of one collide() per worker count, ratio to the previous
    # row and total speed-up over 1 worker
    def table(n, L, Gt, fs):
        rows, t1, prev = [], None, None
        w = 1
        while w <= threads:
            reps = []
            for r in range(3):
                t0 = time.perf_counter()
                O.collide(n, L, Gt, fs[r], 1.0, nthreads=w)
                reps.append(time.perf_counter() - t0)
            t = sorted(reps)[1]
            t1 = t1 or t
            rows.append({"cores": w, "time": t, "ratio": (prev / t) if prev else 1.0, "total_speedup": t1 / t})
            prev = t
            w *= 2
        return {"columns": "cores,time,ratio,total_speedup", "N": n, "L": L, "rows": rows}

    tables = [table(N_VEL, L_VEL, G, cells)]
    del G
    g24 = VelocityGrid.create(24, 8.0)  # cfg4's grid (Tables 2/4 are N=24)
    G24 = O.generate_table(24, 8.0, LAM, nthreads=threads)
    tables.append(table(24, 8.0, G24, scenarios.mixture_cells(g24, 3, seed=4195)))
    del G24
    # N=32 (SURVEY.md §8d asks for N=16 and N=32): the dense table is 8.6 GB of host memory
    g32 = VelocityGrid.create(32, 8.0)
    G32 = O.generate_table(32, 8.0, LAM, nthreads=threads)
    tables.append(table(32, 8.0, G32, scenarios.mixture_cells(g32, 3, seed=4195)))
    del G32
    return {"value": ev / el, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": f"{ev} single-cell collide() evals at N=16 (cfg2 cells 0..63, OpenMP over zeta_k, "
                      f"{threads} threads, {el:.1f} s)",
            "tables_1_4": tables}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1301_4195_b200 import VelocityGrid, scenarios
    O.build()
    threads = os.cpu_count()
    grid = VelocityGrid.create(N_VEL, L_VEL)
    G = O.generate_table(N_VEL, L_VEL, LAM, nthreads=threads)
    sample = 16  # cells per step: one RK2 step (2 evals) of 16 cfg2 cells
    f = scenarios.mixture_cells(grid, sample, seed=4195)
    for _ in range(args.warmup):
        O.collision_rk2(N_VEL, L_VEL, G, f, DT, 1.0, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        f = O.collision_rk2(N_VEL, L_VEL, G, f, DT, 1.0, nthreads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = 2 * sample * args.steps / tot
    line = {
        "impl": "reference", "metric": "collision-operator evals/s (N=16, cfg2 two-Maxwellian cells, RK2)",
        "value": value, "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / PUBLISHED_EVALS_PER_S, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg2 sample: RK2 step of {sample} cells (of 4096), N=16, L=6, lambda=1",
                   "cells_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} cells x {args.steps} RK2 steps, oracle/boltz_oracle.c "
                                   f"(OpenMP over zeta_k, {threads} threads)"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
    from paper_1301_4195_b200.boltz import fp64_peak
    from paper_1301_4195_b200.build import build

    if rank == 0:
        build()
    # one rank per GPU over NCCL; BOLTZ_BENCH_DIST=gloo (CPU collectives, ranks
    # folded onto the visible GPUs) only checks the multi-rank plumbing on a
    # box with fewer GPUs than ranks -- its timings are not bench values
    backend = os.environ.get("BOLTZ_BENCH_DIST", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend == "gloo" else local
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        dist.barrier()
        build()  # no-op unless stale
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # where the timing collectives run
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    grid = VelocityGrid.create(N_VEL, L_VEL)
    t0 = time.perf_counter()
    G = generate_table(grid, KernelSpec(LAM))
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    op = CollisionOperator(grid, KernelSpec(LAM), G, device=local)
    t_upload = time.perf_counter() - t0
    cells = args.cells
    f_host = scenarios.mixture_cells(grid, cells, seed=4195 + 7919 * rank)
    f = torch.from_numpy(f_host).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    peak = fp64_peak(local, 0.5)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        op.collision_rk2(f, DT)
    torch.cuda.synchronize()
    op.timing(reset=True)
    op.set_timing(True)
    stream = torch.cuda.current_stream()
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            op.collision_rk2(f, DT)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        barrier()
    op.set_timing(False)
    kms, klaunch = op.timing(reset=True)
    total_ms = sum(step_ms)
    tmax = torch.tensor([total_ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    evals = 2 * cells * args.steps * world
    value = evals / (total_ms * 1e-3)

    # roofline of the dominant kernel (K2 convolution)
    terms_plain, terms_mirror = op.schedule_terms()
    conv_kernel = "k_conv_mirror<16>" if terms_mirror else "k_conv_pipe<16>"
    exec_ratio = (terms_mirror or terms_plain) / terms_per_eval(N_VEL)
    conv_launches = klaunch["conv"]
    conv_ms_avg = kms["conv"] / max(conv_launches, 1)
    flop_per_launch = FLOP_PER_TERM * terms_per_eval(N_VEL) * cells
    achieved = flop_per_launch / (conv_ms_avg * 1e-3) / 1e12

    # e2e: the public API with HOST buffers (pinned), H2D + compute + D2H every step
    pinned = torch.from_numpy(f_host).pin_memory()
    ph = pinned.numpy()
    for _ in range(1):
        op.collision_rk2(ph, DT)
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op.collision_rk2(ph, DT)  # synchronous: copies in, 2 evals per cell, copies out
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    te = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = evals / (float(te.item()) * 1e-3)

    # N=32 (cfg5-shaped: 2048 two-Maxwellian cells, L=8) sub-measurement
    cfg3 = bench_cfg3(op, dev) if rank == 0 and not args.no_cfg3 else None

    n32 = None
    if not args.no_n32 and rank == 0:
        op.close()
        del G
        n32 = bench_n32(args, dev, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "collision-operator evals/s (N=16, cfg2; FP64)",
            "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": value / PUBLISHED_EVALS_PER_S, "dtype": "f64", "data": "synthetic",
            "vs_baseline_ref": "BASELINE.md: 245.1 evals/s = 1 / 0.00408 s per N=16 eval on 16 Stampede cores "
                               "(PAPER.md:358), other hardware",
            "config": {"workload": f"cfg2: {cells} independent cells per GPU, N=16^3 on [-6,6]^3, hard spheres, "
                                   "one collision RK2 step (2 collide evals) per cell per step",
                       "cells_per_gpu": cells, "N": N_VEL, "L": L_VEL, "lambda": LAM, "dt": DT,
                       "parallelism": f"cells sharded, {world} rank(s), no collective on the data path",
                       "l2": "flushed (256 MiB write) before every timed step; f 128 MiB + fhat 256 MiB > L2"},
            "cells_steps_per_s": value / 2.0,
            "gpu_launches": int(sum(klaunch.values())),
            "kernel_ms": {k: round(v, 4) for k, v in kms.items()},
            "kernel_launches": klaunch,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(conv_kernel, cells),
                         "kernel": f"{conv_kernel} (K2)",
                         "executed_term_ratio": exec_ratio,
                         "executed_fp64_slot_fraction": achieved / peak * exec_ratio * 12 / 10,
                         "note": "achieved = 10 flop x 27/64 N^6 valid terms x cells per launch / mean launch time "
                                 "(algorithmic, SURVEY.md §8d). The kernel executes executed_term_ratio of those "
                                 "terms (pair symmetry, plus the Hermitian mirror of interior terms for collide / "
                                 "RK2, DESIGN.md §2-3; the ratio is the library's folded-table size) at 6 FP64 "
                                 "pipe instructions (2 DMUL + 4 DFMA) each, so the FP64 pipe-slot fraction is frac "
                                 "x executed_term_ratio x 12/10. peak = DFMA probe measured in this run "
                                 "(MEASURED_PEAKS.json has no FP64 entry)"},
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": int(cells * N_VEL ** 3 * 8),
                    "d2h_bytes_per_step": int(cells * N_VEL ** 3 * 8),
                    "path": "CollisionOperator.collision_rk2(pinned numpy) -> boltz_rk2_batch(mem=HOST)"},
            "clocks": clk.summary(),
            "setup_s": {"table_generate": round(t_gen, 3), "table_upload_fold": round(t_upload, 3)},
        }
        if n32:
            line["n32"] = n32
        if cfg3:
            line["cfg3"] = cfg3
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_cfg3(op, dev, steps=60):
    """cfg3 (BASELINE.json configs[2]) on this rank: Nx=256 geometric cells,
    diffuse wall T_w=2, Strang steps (SSP-RK2 transport + RK2 collision) replayed
    as a CUDA graph of 3 steps; 1 rank (the halo path is exercised by tests)."""
    import torch
    from paper_1301_4195_b200 import scenarios
    from paper_1301_4195_b200.solver import Boundary, Solver1D
    grid = op.grid
    x, dx = scenarios.geometric_grid(256, 20.0, 1.02)
    f0 = np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (256, 1))
    op.set_schedule("latency")  # 256 cells: K2 rows split over 4 warps
    s = Solver1D(op, x, dx, f0, left=Boundary("wall", 2.0), right=Boundary("extrap"), device=dev)
    dt = s.cfl_dt()
    s.strang_step(dt)
    op.timing(reset=True)
    s.capture(dt)  # the launches of 3 Strang steps are counted here, at capture
    _, counts = op.timing(reset=True)
    launches_per_step = sum(counts.values()) / 3
    s.advance(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.advance(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    op.set_schedule("throughput")
    return {"workload": "cfg3: Nx=256 geometric (1.02) on [0,20], N=16 L=6, diffuse wall T_w=2, dt=CFL 0.9",
            "steps": steps, "ms_per_step": ms / steps, "cells_steps_per_s": 256 * steps / (ms * 1e-3),
            "evals_per_s": 2 * 256 * steps / (ms * 1e-3),
            "mode": "async library + CUDA graph of 3 Strang steps, K2 latency schedule",
            "launches_per_step": launches_per_step}


def bench_n32(args, dev, local):
    import torch
    from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
    n, L, cells = 32, 8.0, 2048
    grid = VelocityGrid.create(n, L)
    t0 = time.perf_counter()
    G = generate_table(grid, KernelSpec(LAM))
    t_gen = time.perf_counter() - t0
    op = CollisionOperator(grid, KernelSpec(LAM), G, device=local)
    del G
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=4195)).to(dev)
    for _ in range(1):
        op.collision_rk2(f, 1e-3)
    torch.cuda.synchronize()
    op.timing(reset=True)
    op.set_timing(True)
    steps = 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        op.collision_rk2(f, 1e-3)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kms, kl = op.timing(reset=True)
    op.close()
    conv_avg = kms["conv"] / max(kl["conv"], 1)
    # the workspace may split the batch: flops per launch = per-launch cells share
    flop_total = FLOP_PER_TERM * terms_per_eval(n) * cells * 2 * steps
    return {"workload": f"cfg5-shaped: {cells} cells, N=32^3 on [-8,8]^3, lambda=1, RK2 steps",
            "value": 2 * cells * steps / (ms * 1e-3), "unit": "evals/s", "steps": steps, "warmup": 1,
            "ms_per_step": ms / steps, "conv_tflops_algorithmic": flop_total / (kms["conv"] * 1e-3) / 1e12,
            "conv_ms_per_kernel": conv_avg, "conv_kernels_per_eval": kl["conv"] / (2 * steps),
            "table_generate_s": round(t_gen, 2)}


if __name__ == "__main__":
    main()

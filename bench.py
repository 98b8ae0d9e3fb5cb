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
# identical in both arms, so the driver can divide them
METRIC = "collision-operator evals/s (N=16, cfg2 two-Maxwellian cells, RK2 step; FP64)"
# parity witnesses of the timed cfg2 batch: lanes 0 and 31, several 32-cell
# groups, the first and last chunk of the host pipeline (1,3,3,1 x 512 cells)
WITNESS16 = (0, 31, 32, 511, 549, 2047, 2148, 4095)
WITNESS32 = (0, 1234)


def workload_config(cells, world):
    """BASELINE.json configs[1] as this bench runs it (the same dict in both arms)."""
    return {"workload": f"cfg2: {cells} independent cells per GPU, N=16^3 on [-6,6]^3, hard spheres, "
                        "one collision RK2 step (2 collide evals) per cell per step",
            "cells_per_gpu": cells, "N": N_VEL, "L": L_VEL, "lambda": LAM, "dt": DT,
            "seed": "SplitMix64 4195 (+7919 x rank), rho/u/T per mixture component",
            "parallelism": f"cells sharded, {world} rank(s), no collective on the data path",
            "l2": "flushed (256 MiB write) before every timed step; f 128 MiB + fhat 256 MiB > L2"}


def host_cpu():
    """CPU model, physical cores and logical CPUs this process may run on."""
    cpus = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    model, cores, cur = None, set(), {}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh.read().splitlines() + [""]:
                if not line.strip():
                    if cur.get("processor") is not None and int(cur["processor"]) in cpus:
                        cores.add((cur.get("physical id", "0"), cur.get("core id", cur["processor"])))
                    cur = {}
                    continue
                k, _, v = line.partition(":")
                cur[k.strip()] = v.strip()
                if k.strip() == "model name" and model is None:
                    model = v.strip()
    except OSError:
        pass
    return {"cpu_model": model, "physical_cores": len(cores) or len(cpus), "logical_cpus": len(cpus)}


def pin_openmp():
    """The reference's OpenMP run settings: one
    thread per physical core, bound close.  Only for processes that run nothing
    but the CPU oracle: libgomp binds its initial thread when it loads, so
    host_cpu() must be read before, and the GPU arm's own host threads must not
    inherit the binding (the CPU legs run in a subprocess there)."""
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    return f"OMP_PROC_BIND={os.environ['OMP_PROC_BIND']} OMP_PLACES={os.environ['OMP_PLACES']}"


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
    p.add_argument("--cpu-baseline-only", action="store_true", help=argparse.SUPPRESS)
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
def cpu_baseline_subprocess(seconds):
    """cpu_baseline() in a fresh process pinned like the reference's OpenMP run."""
    env = dict(os.environ, OMP_PROC_BIND="close", OMP_PLACES="cores")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-only", "--cpu-seconds",
                        str(seconds)], capture_output=True, text=True, env=env)
    if r.returncode != 0:
        return {"error": r.stderr[-400:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def cpu_baseline(seconds, omp, hw):
    """Oracle port (C, OpenMP over zeta_k) on this host: evals/s at N=16,
    plus the reference's bench_collision tables at N=16/24/32."""
    from oracle import oracle as O
    from paper_1301_4195_b200 import VelocityGrid, scenarios
    O.build()
    threads = hw["physical_cores"]
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
        while True:
            reps = []
            for r in range(3):
                t0 = time.perf_counter()
                O.collide(n, L, Gt, fs[r], 1.0, nthreads=w)
                reps.append(time.perf_counter() - t0)
            t = sorted(reps)[1]
            t1 = t1 or t
            rows.append({"cores": w, "time": t, "ratio": (prev / t) if prev else 1.0, "total_speedup": t1 / t})
            prev = t
            if w == threads:
                break
            w = min(2 * w, threads)
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
            **hw, "omp": omp, "tables_1_4": tables}


def run_reference(args, rank, world, omp, hw):
    """The reference arm: the oracle port of the reference's OpenMP collision
    path on this box's host cores, on a bounded sample of the
    same cfg2 workload, printed under the same metric and config."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1301_4195_b200 import VelocityGrid, scenarios
    O.build()
    threads = hw["physical_cores"]
    grid = VelocityGrid.create(N_VEL, L_VEL)
    G = O.generate_table(N_VEL, L_VEL, LAM, nthreads=threads)
    sample = 16  # cells per step: one RK2 step (2 evals) of 16 of the 4096 cfg2 cells
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
    desc = (f"{sample} of the {args.cells} cfg2 cells per step (cells 0..{sample - 1}), RK2 step = 2 evals per "
            f"cell; evals/s is the per-eval rate, which is batch-size independent on the CPU (cells run one "
            f"after another, OpenMP over zeta_k inside each eval)")
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / PUBLISHED_EVALS_PER_S, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.cells, world),
        "sample": desc,
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": f"{desc}; oracle/boltz_oracle.c, {threads} threads", **hw, "omp": omp},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def main():
    args = parse()
    hw = host_cpu()  # before libgomp can bind this thread
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.cpu_baseline_only:
        print(json.dumps(cpu_baseline(args.cpu_seconds, pin_openmp(), hw)), flush=True)
        return
    if args.impl == "reference":
        return run_reference(args, rank, world, pin_openmp(), hw)
    if world > 1:  # communicator init lines (ranks, transport) on stderr for the driver's check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

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
    wit = [c for c in WITNESS16 if c < cells]

    peak = fp64_peak(local, 0.5)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(step, nsteps, before_last=None):
        """nsteps device-timed calls of step(), L2 flushed and ranks aligned
        before each; before_last() runs (untimed) ahead of the last one."""
        ms = []
        for i in range(nsteps):
            flush.zero_()  # L2 flush outside the timed events
            if i == nsteps - 1 and before_last:
                before_last()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        barrier()
        return ms

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        op.collision_rk2(f, DT)
    torch.cuda.synchronize()
    op.timing(reset=True)
    op.set_timing(True)
    snap = {}
    with ClockSampler(local) as clk:
        step_ms = timed(lambda: op.collision_rk2(f, DT), args.steps,
                        before_last=lambda: snap.update(dev=f[wit].cpu().numpy()))
    op.set_timing(False)
    kms, klaunch = op.timing(reset=True)
    total_ms = max_over_ranks(sum(step_ms))
    evals = 2 * cells * args.steps * world
    value = evals / (total_ms * 1e-3)
    dev_after = f[wit].cpu().numpy()

    # roofline of the dominant kernel (K2 convolution)
    terms_plain, terms_mirror = op.schedule_terms()
    conv_kernel = f"{op.conv_kernel()}<{N_VEL}>"
    exec_ratio = (terms_mirror or terms_plain) / terms_per_eval(N_VEL)
    conv_launches = klaunch["conv"]
    conv_ms_avg = kms["conv"] / max(conv_launches, 1)
    flop_per_launch = FLOP_PER_TERM * terms_per_eval(N_VEL) * cells
    achieved = flop_per_launch / (conv_ms_avg * 1e-3) / 1e12
    # nominal FP64 peak at the sampled SM clock: 148 SMs x 64 DFMA/clk x 2 flop
    sm_mhz = clk.summary()["sm_mhz"] or 1965.0
    peak_nominal = torch.cuda.get_device_properties(dev).multi_processor_count * 64 * 2 * sm_mhz * 1e6 / 1e12

    # e2e: the public API with HOST buffers, H2D + compute + D2H every step;
    # pinned (the library's pipeline overlaps copies with compute) and pageable
    # (plain numpy / std::vector memory, what the reference's caller holds)
    pinned = torch.from_numpy(f_host).pin_memory()
    ph = pinned.numpy()
    for _ in range(args.warmup):
        op.collision_rk2(ph, DT)
    e2e_ms = timed(lambda: op.collision_rk2(ph, DT), args.steps,
                   before_last=lambda: snap.update(e2e=ph[wit].copy()))
    e2e_value = evals / (max_over_ranks(sum(e2e_ms)) * 1e-3)
    pg = f_host.copy()
    for _ in range(args.warmup):
        op.collision_rk2(pg, DT)
    pg_ms = timed(lambda: op.collision_rk2(pg, DT), args.steps)
    pg_value = evals / (max_over_ranks(sum(pg_ms)) * 1e-3)
    pageable_bitwise = bool(np.array_equal(pg, ph))

    # parity witness: the last timed step of sampled cells against the oracle's
    # collision_rk2 with the same host table G (SURVEY.md §8c bar: 1e-10)
    parity = None
    if rank == 0:
        from oracle import oracle as O
        O.build()
        th = hw["physical_cores"]
        r_dev = O.collision_rk2(N_VEL, L_VEL, G, snap["dev"], DT, 1.0, nthreads=th)
        r_e2e = O.collision_rk2(N_VEL, L_VEL, G, snap["e2e"], DT, 1.0, nthreads=th)

        def rel(got, ref, before):
            return max(float(np.abs(g - r).max() / max(np.abs(r - b).max(), 1e-300))
                       for g, r, b in zip(got, ref, before))
        parity = {"cells": wit, "reference": "oracle collision_rk2 (same host G), last timed step",
                  "max_rel_increment_n16_device": rel(dev_after, r_dev, snap["dev"]),
                  "max_rel_increment_n16_e2e": rel(ph[wit], r_e2e, snap["e2e"]),
                  "max_rel_state_n16": max(rel_state(dev_after, r_dev), rel_state(ph[wit], r_e2e))}

    # cfg3 (Strang steps with the halo); on N>1 ranks strong-scaled with NCCL halo.
    # A failure here is reported in the line, not allowed to lose the headline.
    cfg3 = None
    if not args.no_cfg3:
        try:
            cfg3 = bench_cfg3(op, dev, rank, world, backend)
        except Exception as exc:  # noqa: BLE001
            cfg3 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            op.set_schedule("throughput")

    cfg1 = None
    if rank == 0 and not args.no_cfg3:
        try:
            cfg1 = bench_cfg1(op, dev)
        except Exception as exc:  # noqa: BLE001
            cfg1 = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    n32 = None
    if not args.no_n32 and rank == 0:
        op.close()
        del G
        n32 = bench_n32(args, dev, local, hw)
        if parity is not None and n32.get("parity"):
            parity.update(n32.pop("parity"))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_subprocess(args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": value / PUBLISHED_EVALS_PER_S, "dtype": "f64", "data": "synthetic",
            "vs_baseline_ref": "BASELINE.md: 245.1 evals/s = 1 / 0.00408 s per N=16 eval on 16 Stampede cores "
                               "(PAPER.md:358), other hardware",
            "config": workload_config(cells, world),
            "cells_steps_per_s": value / 2.0,
            "gpu_launches": int(sum(klaunch.values())),
            "kernel_ms": {k: round(v, 4) for k, v in kms.items()},
            "kernel_launches": klaunch,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(conv_kernel, cells),
                         "peak_source": "builder-probed: k_dfma_probe (32 warps/SM x 8 independent DFMA chains) "
                                        "timed in this run; MEASURED_PEAKS.json has no FP64 entry",
                         "peak_nominal": peak_nominal,
                         "frac_nominal": achieved / peak_nominal,
                         "peak_nominal_source": "148 SMs x 64 DFMA/clk x 2 flop x median sampled SM clock",
                         "kernel": f"{conv_kernel} (K2)",
                         "executed_term_ratio": exec_ratio,
                         "executed_fp64_slot_fraction": achieved / peak * exec_ratio * 12 / 10,
                         "executed_fp64_slot_fraction_nominal": achieved / peak_nominal * exec_ratio * 12 / 10,
                         "note": "achieved = 10 flop x 27/64 N^6 valid terms x cells per launch / mean launch time "
                                 "(algorithmic, SURVEY.md §8d). The kernel executes executed_term_ratio of those "
                                 "terms (pair symmetry, plus the Hermitian mirror of interior terms for collide / "
                                 "RK2, DESIGN.md §2-3; the ratio is the library's folded-table size) at 6 FP64 "
                                 "pipe instructions (2 DMUL + 4 DFMA) each, so frac > 1 is exact work avoided, "
                                 "and the hardware FP64 pipe-slot fraction is frac x executed_term_ratio x 12/10"},
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": int(cells * N_VEL ** 3 * 8),
                    "d2h_bytes_per_step": int(cells * N_VEL ** 3 * 8),
                    "path": "CollisionOperator.collision_rk2(pinned numpy) -> boltz_rk2_batch(mem=HOST)"},
            "e2e_pageable": {"value": pg_value, "unit": "evals/s", "h2d_bytes_per_step": int(cells * N_VEL ** 3 * 8),
                             "d2h_bytes_per_step": int(cells * N_VEL ** 3 * 8),
                             "ratio_to_pinned": pg_value / e2e_value, "bitwise_equal_to_pinned": pageable_bitwise,
                             "path": "CollisionOperator.collision_rk2(plain numpy) -> boltz_rk2_batch(mem=HOST)"},
            "clocks": clk.summary(),
            "setup_s": {"table_generate": round(t_gen, 3), "table_upload_fold": round(t_upload, 3)},
        }
        if parity:
            line["parity"] = parity
        if n32:
            line["n32"] = n32
        if cfg3:
            line["cfg3"] = cfg3
        if cfg1:
            line["cfg1"] = cfg1
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def rel_state(got, ref):
    return max(float(np.abs(g - r).max() / max(np.abs(r).max(), 1e-300)) for g, r in zip(got, ref))


class _HostStagedHalo:
    """BOLTZ_BENCH_DIST=gloo plumbing check only: the field goes through host
    memory to torch.distributed gloo P2P (ranks folded onto one GPU cannot share
    an NCCL communicator).  Not a measurement path."""

    def __init__(self, rank, world):
        from paper_1301_4195_b200.solver import TorchHalo
        self.h = TorchHalo(rank, world)

    def exchange(self, field):
        host = field.cpu()
        n = self.h.exchange(host)
        field.copy_(host)
        return n


def bench_cfg3(op, dev, rank, world, backend, steps=60):
    """cfg3 (BASELINE.json configs[2]): Nx=256 geometric cells, diffuse wall
    T_w=2, Strang steps (SSP-RK2 transport + RK2 collision).  One rank: CUDA
    graph of 3 Strang steps.  N>1 ranks: STRONG-scaled -- the 256 cells are
    sharded by plan_decomposition and the ghosts cross ranks through the
    library's NCCL halo (boltz_halo_exchange, captured in the same graph);
    rank 0 then recomputes the run unsharded and compares bitwise (the
    decomposition transparency contract)."""
    import torch
    import torch.distributed as dist
    from paper_1301_4195_b200 import NcclHalo, scenarios
    from paper_1301_4195_b200.solver import Boundary, Solver1D, k2_schedule, plan_decomposition
    grid = op.grid
    nx = 256
    x, dx = scenarios.geometric_grid(nx, 20.0, 1.02)
    m0 = scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0)
    init = lambda start, count: np.tile(m0, (count, 1))  # noqa: E731
    # K2 rows split into fixed segments: 4 (<= 256 cells per rank) or 8 (<= 64: the 8-rank shard); one schedule for
    # every rank and for the one-rank recomputation, so bitwise_vs_1rank holds
    sched = k2_schedule(grid.n, max(c for _, c in plan_decomposition(nx, world)))
    op.set_schedule(sched)
    kw = dict(left=Boundary("wall", 2.0), right=Boundary("extrap"), device=dev)
    halo = None
    if world > 1:
        halo = NcclHalo(rank, world, dev.index) if backend == "nccl" else _HostStagedHalo(rank, world)
    # NCCL halo: the exchange overlaps the ghost-free rows of each transport stage
    s = Solver1D(op, x, dx, init, rank=rank, world=world, halo=halo, overlap_halo=isinstance(halo, NcclHalo), **kw)
    dt = s.cfl_dt()
    graph = world == 1 or isinstance(halo, NcclHalo)
    s.strang_step(dt)  # warm-up: workspace + kernel attributes
    op.timing(reset=True)
    if graph:
        s.capture(dt)  # the launches of 3 Strang steps are counted here, at capture
        _, counts = op.timing(reset=True)
        launches_per_step = sum(counts.values()) / 3
        s.advance(3)
    else:
        launches_per_step = None
        for _ in range(3):
            s.strang_step(dt)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graph:
        s.advance(steps)
    else:
        for _ in range(steps):
            s.strang_step(dt)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64,
                      device=dev if backend == "nccl" else torch.device("cpu"))
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    done = 1 + 3 + steps  # Strang steps each rank has taken
    out = {"workload": "cfg3: Nx=256 geometric (1.02) on [0,20], N=16 L=6, diffuse wall T_w=2, dt=CFL 0.9",
           "ranks": world, "scaling": "strong" if world > 1 else None, "steps": steps, "ms_per_step": ms / steps,
           "cells_steps_per_s": nx * steps / (ms * 1e-3), "evals_per_s": 2 * nx * steps / (ms * 1e-3),
           "mode": ("CUDA graph of 3 Strang steps" if graph else "eager Strang steps") + f", K2 {sched} schedule"
                   + (", NCCL halo (boltz_halo_exchange) inside the graph, overlapped with the ghost-free rows"
                      if isinstance(halo, NcclHalo) else
                      ", host-staged gloo halo (plumbing check, not a measurement)" if world > 1 else ""),
           "launches_per_step_rank0": launches_per_step}
    if world > 1:
        n3 = grid.size()
        # 4 ghost refreshes per Strang step (2 sub-steps x 2 stages), 2 cells x N^3 doubles each way per boundary
        out["halo_bytes_per_step"] = {"per_boundary_each_way": 4 * 2 * n3 * 8,
                                      "total": 4 * 2 * 2 * (world - 1) * n3 * 8}
        parts = [None] * world if rank == 0 else None
        dist.gather_object((s.start, s.interior.cpu().numpy()), parts, dst=0)
        # every rank tears the communicator down here, together and in order: the graph that holds the
        # captured exchanges first, then ncclCommDestroy (which waits for such graphs, and for the peers)
        s.release_graph()
        if isinstance(halo, NcclHalo):
            halo.close()
        if rank == 0:
            parts.sort(key=lambda p: p[0])
            sharded = np.concatenate([p[1] for p in parts])
            one = Solver1D(op, x, dx, init, rank=0, world=1, halo=None, **kw)
            one.strang_step(dt)
            one.run(dt, done - 1, graph=True)
            out["bitwise_vs_1rank"] = bool(np.array_equal(sharded, one.interior.cpu().numpy()))
            out["steps_compared"] = done
    op.set_schedule("throughput")
    return out


def bench_cfg1(op, dev, steps=50):
    """cfg1 (BASELINE.json configs[0]): one cell, N=16, the two-Maxwellian
    state with noise, 50 RK2 steps of dt = 0.01 -- K2 in the cell schedule
    (lane = output k3), one RK2 step captured in a CUDA graph and replayed."""
    import torch
    from paper_1301_4195_b200 import scenarios
    f0 = scenarios.config1_initial(op.grid)
    f = torch.from_numpy(f0.reshape(1, -1).copy()).to(dev)
    op.set_schedule("cell")
    try:
        op.collision_rk2(f, 0.01)  # warm-up: workspace, attributes
        op.set_async(True)
        st = torch.cuda.Stream(dev)
        st.wait_stream(torch.cuda.current_stream(dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                op.collision_rk2(f, 0.01)
        torch.cuda.current_stream(dev).wait_stream(st)
        for _ in range(3):
            g.replay()
        op.sync()
        f.copy_(torch.from_numpy(f0.reshape(1, -1)).to(dev))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        op.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    finally:
        op.set_async(False)
        op.set_schedule("throughput")
    return {"workload": "cfg1: one cell, N=16^3 on [-6,6]^3, hard spheres, 50 RK2 steps of dt=0.01",
            "steps": steps, "ms": ms, "evals_per_s": 2 * steps / (ms * 1e-3),
            "mode": "K2 cell schedule (lane = output k3), CUDA graph of one RK2 step replayed"}


def bench_n32(args, dev, local, hw):
    """cfg5-shaped N=32 sub-measurement: 2048 mixture cells, RK2 steps, with a
    parity witness of two cells of the last timed step against the oracle."""
    import torch
    from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
    n, L, cells = 32, 8.0, 2048
    warm, steps = max(3, args.warmup), max(5, min(args.steps, 8))
    grid = VelocityGrid.create(n, L)
    t0 = time.perf_counter()
    G = generate_table(grid, KernelSpec(LAM))
    t_gen = time.perf_counter() - t0
    op = CollisionOperator(grid, KernelSpec(LAM), G, device=local)
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=4195)).to(dev)
    for _ in range(warm):
        op.collision_rk2(f, 1e-3)
    torch.cuda.synchronize()
    op.timing(reset=True)
    op.set_timing(True)
    ms = 0.0
    wit = list(WITNESS32)
    snap = None
    step_ms = []
    with ClockSampler(local) as clk:
        for i in range(steps):
            if i == steps - 1:
                snap = f[wit].cpu().numpy()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.collision_rk2(f, 1e-3)
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    ms = sum(step_ms)
    kms, kl = op.timing(reset=True)
    after = f[wit].cpu().numpy()
    op.close()
    from oracle import oracle as O
    O.build()
    ref = O.collision_rk2(n, L, G, snap, 1e-3, 1.0, nthreads=hw["physical_cores"])
    del G
    conv_avg = kms["conv"] / max(kl["conv"], 1)
    flop_total = FLOP_PER_TERM * terms_per_eval(n) * cells * 2 * steps
    return {"workload": f"cfg5-shaped: {cells} cells, N=32^3 on [-8,8]^3, lambda=1, RK2 steps (dt=1e-3)",
            "value": 2 * cells * steps / (ms * 1e-3), "unit": "evals/s", "steps": steps, "warmup": warm,
            "ms_per_step": ms / steps, "conv_tflops_algorithmic": flop_total / (kms["conv"] * 1e-3) / 1e12,
            "conv_ms_per_kernel": conv_avg, "conv_kernels_per_eval": kl["conv"] / (2 * steps),
            "table_generate_s": round(t_gen, 2), "step_ms": [round(x, 2) for x in step_ms], "clocks": clk.summary(),
            "parity": {"cells_n32": wit,
                       "max_rel_increment_n32": max(float(np.abs(a - r).max() / max(np.abs(r - b).max(), 1e-300))
                                                    for a, r, b in zip(after, ref, snap)),
                       "max_rel_state_n32": rel_state(after, ref)}}


if __name__ == "__main__":
    main()

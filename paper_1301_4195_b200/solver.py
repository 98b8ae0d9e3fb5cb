"""Space-inhomogeneous driver: Strang splitting of second-order FV transport
and the GPU collision RK2, with the spatial domain sharded across ranks
(SPEC.md:372-481).

    strang_step(dt) = T(dt/2) o C_RK2(dt) o T(dt/2)
    T(h): SSP-RK2 (Heun) of the explicit FV step S:
          t1 = S(f), f <- f/2 + S(t1)/2, each S after a ghost refresh (halo
          exchange / wall / extrapolation) -- DESIGN.md §5 item 4.  The SPEC's
          literal single stage, f <- S(f) with one ghost refresh
          (SPEC.md:342-345,471), is `transport_scheme="single_stage"`.
    C_RK2(dt): boltz_rk2_batch over the rank's interior cells -- cell-local,
          no communication

Decomposition: contiguous cell ranges balanced to +-1.
Halo: each transport sub-step refreshes 2 ghost cells per side
(SPEC.md:296,448,471); the two edge cells of a rank are one contiguous
2*N^3 block, so one send + one recv per neighbour (grouped P2P via
torch.distributed -- NCCL over NVLink on GPUs, gloo on CPU), with no
even/odd ordering needed.  LoopbackHalo runs n virtual
ranks in one process (the SPEC's required in-process backend).

The field layout is the reference's DistributionField: (n_local + 4) x N^3,
ghosts at 0,1 and n_local+2, n_local+3.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .boltz import CollisionOperator, ConfigError, NcclHalo, NumericError
from .scenarios import extend_ghosts


def plan_decomposition(ncells: int, nranks: int) -> List[Tuple[int, int]]:
    """(start, count) per rank; contiguous, ordered, |count_r - count_s| <= 1,
    larger ranges first.  More ranks than cells -> error."""
    if nranks < 1 or ncells < nranks:
        raise ConfigError(f"plan_decomposition: {nranks} ranks for {ncells} cells")
    base, rem = divmod(ncells, nranks)
    out, s = [], 0
    for r in range(nranks):
        c = base + (1 if r < rem else 0)
        out.append((s, c))
        s += c
    return out


def k2_schedule(n: int, cells_per_rank: int) -> str:
    """The K2 schedule for a rank's collision batch (CollisionOperator.set_schedule).
    Small batches at N <= 16 split each row's entries into fixed segments:
    8 up to 64 cells, 4 up to 256 (B200, ms per RK2 step, schedules 1 / 2:
    32 cells 0.235 / 0.196, 64 cells 0.296 / 0.291, 128 cells 0.491 / 0.500,
    256 cells 0.893 / 0.914; `scripts/dev/sched_sweep.py`).  Every rank of a run
    must use the same schedule for the decomposition to stay bitwise transparent
    (SPEC.md:465), so callers pick it from the largest rank's cell count."""
    if n <= 16 and cells_per_rank <= 64:
        return "latency8"
    if n <= 16 and cells_per_rank <= 256:
        return "latency"
    return "throughput"


def predict_speedup(n: int, p: int, N: int, M: int, T_mem: float, T_flop: float, C: float) -> float:
    """The paper's leading-order speed-up model of the decomposed solver
    (§4.2; reference SPEC.md:454-462): n processes of p cores, N^3
    velocity nodes, M cells, halo cost 4 n N^3 T_mem against C M N^6 T_flop of
    collision work,
        S = C M N^6 T_flop / (4 n N^3 T_mem + C M N^6 T_flop / (n p)).
    T_mem = 0 gives exactly n p."""
    if min(n, p, N, M, C, T_flop) <= 0 or T_mem < 0:
        raise ConfigError("predict_speedup: all arguments must be positive (T_mem >= 0)")
    work = C * M * float(N) ** 6 * T_flop
    return work / (4.0 * n * float(N) ** 3 * T_mem + work / (n * p))


@dataclass
class Boundary:
    """Physical end condition: kind 'extrap' (linear extrapolation,
    SPEC.md:318), 'wall' (diffuse Maxwell wall, continuum
    sigma_w as in the reference) or 'wall_balanced' (extension: the same wall
    with sigma_w from the discrete flux balance -- zero net wall mass flux)."""
    kind: str = "extrap"
    Tw: float = 1.0
    Vw: Tuple[float, float, float] = (0.0, 0.0, 0.0)

    _CODES = {"extrap": 0, "wall": 1, "wall_balanced": 2}

    def code(self) -> int:
        if self.kind not in self._CODES:
            raise ConfigError(f"unknown boundary kind {self.kind!r}")
        return self._CODES[self.kind]

    @property
    def is_wall(self) -> bool:
        return self.code() != 0


class TorchHalo:
    """Two-ghost-cell exchange with the left/right neighbour ranks over
    torch.distributed (NCCL on GPUs, gloo on CPU).  Works on any (ncl+4, M)
    tensor whose rows are cells."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, field) -> int:
        import torch.distributed as dist
        ncl = field.shape[0] - 4
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, field[2:4].contiguous(), self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, field[0:2], self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, field[ncl:ncl + 2].contiguous(), self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, field[ncl + 2:ncl + 4], self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return len(ops) // 2


class LoopbackHalo:
    """In-process backend over a list of per-rank fields."""

    @staticmethod
    def exchange_all(fields: Sequence) -> None:
        for r in range(len(fields) - 1):
            a, b = fields[r], fields[r + 1]
            ncl = a.shape[0] - 4
            a[ncl + 2:ncl + 4] = b[2:4]   # right ghosts of r = first two interior of r+1
            b[0:2] = a[ncl:ncl + 2]       # left ghosts of r+1 = last two interior of r


class Solver1D:
    """One rank's share of a 1D-in-space kinetic problem on the GPU.

    x, dx: global cell centres / widths (Nx); f0: global initial field
    (Nx, N^3) or a callable(start, count) -> (count, N^3) (so ranks only
    build their own cells).
    """

    def __init__(self, op: CollisionOperator, x: np.ndarray, dx: np.ndarray, f0, *, rank: int = 0,
                 world: int = 1, left: Boundary = Boundary(), right: Boundary = Boundary(),
                 epsilon: float = 1.0, halo=None, device=None, plan=None, transport_scheme: str = "ssp_rk2",
                 overlap_halo: bool = False):
        import torch
        if transport_scheme not in ("ssp_rk2", "single_stage"):
            raise ConfigError(f"transport_scheme must be 'ssp_rk2' or 'single_stage', got {transport_scheme!r}")
        self.scheme = transport_scheme
        self.overlap_halo = overlap_halo
        self._side = None
        self.op, self.rank, self.world, self.eps = op, rank, world, epsilon
        self.left, self.right = left, right
        self.n3 = op.grid.size()
        plan = plan or plan_decomposition(len(x), world)
        self.start, self.ncl = plan[rank]
        if self.ncl < 2:
            raise ConfigError("each rank needs at least 2 cells (2-cell halo, SPEC.md:438)")
        xe, dxe = extend_ghosts(np.asarray(x, float), np.asarray(dx, float))
        self.x_glob, self.dx_glob = np.asarray(x, float), np.asarray(dx, float)
        sl = slice(self.start, self.start + self.ncl + 4)
        self.device = device if device is not None else torch.device("cuda", op.device)
        self.x_ext = torch.from_numpy(xe[sl].copy()).to(self.device)
        self.dx_ext = torch.from_numpy(dxe[sl].copy()).to(self.device)
        self.field = torch.zeros((self.ncl + 4, self.n3), dtype=torch.float64, device=self.device)
        init = f0(self.start, self.ncl) if callable(f0) else np.asarray(f0)[self.start:self.start + self.ncl]
        self.field[2:self.ncl + 2] = torch.from_numpy(np.ascontiguousarray(init, dtype=np.float64)).to(self.device)
        self._tmp = torch.empty_like(self.field)
        self._tmp2 = torch.empty_like(self.field)
        self.halo = halo if halo is not None else (TorchHalo(rank, world) if world > 1 else None)
        self.is_left_end = rank == 0
        self.is_right_end = rank == world - 1
        self.sigma_w = {}
        self.t = 0.0

    @property
    def interior(self):
        return self.field[2:self.ncl + 2]

    def moments(self):
        """(n_local, 7) device tensor: rho, rho V (3), rho e, T, H per interior cell (GPU)."""
        return self.op.moments(self.interior)

    def marginals(self, cells: Optional[Sequence[int]] = None):
        """(len(cells), N) device tensor of marginal_distribution g(v1) for the
        given LOCAL interior cell indices (all interior cells by default; GPU)."""
        rows = self.interior if cells is None else self.interior[list(cells)]
        return self.op.marginal(rows)

    def ledger(self):
        """Global (mass, x-momentum, energy) = sum_j dx_j (rho, rho V1, rho e)_j over all
        ranks -- the conservation ledger of SPEC.md:403 (collision conserves it to
        round-off; transport changes it only by boundary fluxes)."""
        import torch
        m = self.moments()
        dx = self.dx_ext[2:self.ncl + 2]
        tot = torch.stack([(m[:, 0] * dx).sum(), (m[:, 1] * dx).sum(), (m[:, 4] * dx).sum()])
        if self.world > 1:
            if hasattr(self.halo, "all_reduce"):
                self.halo.all_reduce(tot)
            else:
                import torch.distributed as dist
                dist.all_reduce(tot)
        return tot.cpu().numpy()

    def cfl_dt(self, cfl: float = 0.9) -> float:
        """dt <= cfl * min dx / L; global min."""
        return cfl * float(self.dx_glob.min()) / self.op.grid.half_width

    def fill_ghosts(self, exchange: bool = True) -> None:
        if exchange and self.halo is not None:
            self.halo.exchange(self.field)
        self._fill_physical()

    def _fill_physical(self) -> None:
        if self.is_left_end:
            self.sigma_w[0] = self.op.fill_boundary(self.field, self.x_ext, 0, self.left.code(), self.left.Tw,
                                                    self.left.Vw)
        if self.is_right_end:
            self.sigma_w[1] = self.op.fill_boundary(self.field, self.x_ext, 1, self.right.code(), self.right.Tw,
                                                    self.right.Vw)

    def _walls(self):
        return (self.is_left_end and self.left.is_wall, self.is_right_end and self.right.is_wall)

    @property
    def transport_stages(self) -> int:
        return 1 if self.scheme == "single_stage" else 2

    def transport_stage(self, stage: int, dt: float, exchange: bool = True) -> None:
        """Stage of the transport sub-step.  SSP-RK2: stage 0: t1 = S(f);
        stage 1: f <- f/2 + S(t1)/2.  single_stage: stage 0
        is f <- S(f).  S = one FV step after a ghost refresh
        of its input."""
        wl, wr = self._walls()
        if self.scheme == "single_stage":
            self._refresh_and_step(self._tmp, dt, wl, wr, exchange)
            self.field, self._tmp = self._tmp, self.field
            return
        if stage == 0:
            self._refresh_and_step(self._tmp, dt, wl, wr, exchange)
        else:
            self.field, self._tmp = self._tmp, self.field  # field = t1, _tmp = f^n
            out = self._tmp2
            self._refresh_and_step(out, dt, wl, wr, exchange, base=self._tmp, alpha=0.5)
            self._tmp2 = self.field
            self.field = out

    def _refresh_and_step(self, out, dt, wl, wr, exchange, base=None, alpha=0.0) -> None:
        """Ghost refresh of self.field, then out = [alpha base + (1-alpha)] S(field).
        With overlap_halo (NcclHalo, >= 6 cells per rank) the exchange runs on a
        side stream while the rows that read no ghost ([4, ncl)) are updated,
        and the four edge rows follow once it has landed: bitwise the same rows
        (boltz_transport_step_range), the exchange hidden behind the interior
        update."""
        args = (self.x_ext, self.dx_ext, dt, wl, wr)
        if not (exchange and self.overlap_halo and isinstance(self.halo, NcclHalo) and self.ncl >= 6):
            self.fill_ghosts(exchange)
            self._track_flux(dt, wl, wr)
            self.op.transport_step(self.field, out, *args, base=base, alpha=alpha)
            return
        import torch
        main = torch.cuda.current_stream(self.device)
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        self._side.wait_stream(main)
        with torch.cuda.stream(self._side):
            self.halo.exchange(self.field)
        self._fill_physical()  # the physical ends' ghost rows: disjoint from the exchanged ones
        self.op.transport_step(self.field, out, *args, base=base, alpha=alpha, rows=(4, self.ncl))
        main.wait_stream(self._side)
        self._track_flux(dt, wl, wr)  # reads the end faces, whose ghosts may have come over the halo
        self.op.transport_step(self.field, out, *args, base=base, alpha=alpha, rows=(2, 4))
        self.op.transport_step(self.field, out, *args, base=base, alpha=alpha, rows=(self.ncl, self.ncl + 2))

    def track_boundary_flux(self, enable: bool = True) -> None:
        """Accumulate the end-face fluxes of every FV stage (boltz_end_flux) so
        that ledger() + boundary_flux() is conserved to round-off: the
        "ledger vs wall-flux integral" of the reference RunRecord."""
        import torch
        self._flux = torch.zeros(5, dtype=torch.float64, device=self.device) if enable else None

    def boundary_flux(self):
        """Integrated outflow (mass, momentum 1, energy) through the physical ends
        since track_boundary_flux(), summed over ranks (collective)."""
        import torch
        f = self._flux[[0, 1, 4]].clone()
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(f)
        return f.cpu().numpy()

    def _track_flux(self, dt: float, wl: bool, wr: bool) -> None:
        # SSP-RK2: f^{n+1} = f^n - dt/2 (D(f^n) + D(t1)), so each stage's face fluxes weigh dt/2;
        # the single stage weighs its one set of fluxes dt
        if getattr(self, "_flux", None) is not None:
            w = dt if self.scheme == "single_stage" else 0.5 * dt
            self.op.end_flux(self.field, self.x_ext, self.dx_ext, self._flux, w, wl, wr)

    def transport(self, dt: float, exchange: bool = True) -> None:
        """Transport sub-step T(dt): SSP-RK2 of the FV step, or
        the SPEC's single stage (transport_scheme="single_stage")."""
        if dt * self.op.grid.half_width > float(self.dx_glob.min()) * (1 + 1e-12):
            raise ConfigError("transport: CFL violated (dt * L > min dx)")
        for stage in range(self.transport_stages):
            self.transport_stage(stage, dt, exchange)

    def collide(self, dt: float) -> None:
        interior = self.field[2:self.ncl + 2]  # contiguous rows -> in place on device
        self.op.collision_rk2(interior, dt, self.eps)

    def strang_step(self, dt: float) -> None:
        self.transport(0.5 * dt)
        self.collide(dt)
        self.transport(0.5 * dt)
        self.t += dt

    def run(self, dt: float, steps: int, graph: bool = True) -> None:
        """`steps` Strang steps with the device queue kept full: the library runs
        asynchronously (boltz_set_async) and, on a single rank or with the
        NcclHalo (whose NCCL calls are captured), three steps are captured once
        in a CUDA graph and replayed (three steps return the field / scratch
        buffer rotation to its start).  Numeric errors are reported once, at
        the end (boltz_sync)."""
        capturable = self.world == 1 or isinstance(self.halo, NcclHalo)  # torch P2P is not captured
        if not graph or not capturable or steps < 4:
            self.op.set_async(True)
            try:
                for _ in range(steps):
                    self.strang_step(dt)
                self.op.sync()
            finally:
                self.op.set_async(False)
            return
        self.strang_step(dt)  # warm-up outside capture: workspace + kernel attributes
        self.capture(dt)
        self.advance(steps - 1)

    def capture(self, dt: float, capture_error_mode: Optional[str] = None) -> None:
        """Capture three Strang steps of size dt into a CUDA graph (not executed).
        capture_error_mode: torch.cuda.graph's; default "global" on one rank,
        "thread_local" on several."""
        import torch
        self.op.set_async(True)
        stream = torch.cuda.Stream(self.device)
        stream.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        ptrs = [t.data_ptr() for t in (self.field, self._tmp, self._tmp2)]
        t0 = self.t
        # multi-rank: NCCL's own helper threads may make CUDA calls while this thread captures;
        # thread-local capture mode keeps those from invalidating the capture
        mode = capture_error_mode or ("thread_local" if self.world > 1 else "global")
        try:
            with torch.cuda.stream(stream):
                with torch.cuda.graph(g, stream=stream, capture_error_mode=mode):
                    for _ in range(3):
                        self.strang_step(dt)
        finally:
            self.op.set_async(False)
        assert [t.data_ptr() for t in (self.field, self._tmp, self._tmp2)] == ptrs, "buffer rotation"
        torch.cuda.current_stream(self.device).wait_stream(stream)
        self.t = t0
        self._graph, self._graph_dt = g, dt

    def advance(self, steps: int) -> None:
        """`steps` Strang steps of the captured dt: graph replays + eager remainder."""
        g, dt = self._graph, self._graph_dt
        self.op.set_async(True)
        try:
            for _ in range(steps // 3):
                g.replay()
                self.t += 3 * dt
            for _ in range(steps % 3):
                self.strang_step(dt)
            self.op.sync()
        finally:
            self.op.set_async(False)
        self.graph_replays = getattr(self, "graph_replays", 0) + steps // 3

    def release_graph(self) -> None:
        """Drop the captured graph (after the device has drained).  Call it on
        every rank BEFORE closing an NcclHalo whose exchanges the graph holds:
        NCCL keeps a communicator alive, and ncclCommDestroy waiting, while a
        captured graph still references it."""
        import torch
        torch.cuda.synchronize(self.device)
        self._graph = None
        self._graph_dt = None


def strang_step_loopback(solvers: Sequence[Solver1D], dt: float) -> None:
    """One Strang step of n virtual ranks in one process (LoopbackHalo)."""
    for half in (0, 1):
        for stage in range(solvers[0].transport_stages):
            if stage == 1:  # the stage-1 input t1 lives in _tmp until transport_stage swaps it in
                LoopbackHalo.exchange_all([s._tmp for s in solvers])
            else:
                LoopbackHalo.exchange_all([s.field for s in solvers])
            for s in solvers:
                s.transport_stage(stage, 0.5 * dt, exchange=False)
        if half == 0:
            for s in solvers:
                s.collide(dt)
    for s in solvers:
        s.t += dt

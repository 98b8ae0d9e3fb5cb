"""RunRecord: per-output-time moment tables, marginals and the conservation
ledger of a Solver1D run, written as plot-ready CSV (reference SPEC.md cli_io
module: RunRecord, write_moment_csv / write_marginal_csv).

    moments CSV:   t, x_center, dx, rho, V1, T, H            (one row per cell)
    marginals CSV: t, cell_index, v1, g                       (N rows per cell)
    ledger CSV:    t, mass, momentum1, energy, wall_flux_mass

Numbers are written with 17 significant digits, so reading a file back gives
the in-memory doubles exactly (SPEC: "fixed 17-significant-digit decimal
formatting for bit-stable golden files").  All quantities are computed on the
GPU (Solver1D.moments / marginals / ledger); only the per-output rows cross to
the host.  With several ranks, rank 0 gathers the rows (torch.distributed);
other ranks record nothing.
"""
from __future__ import annotations

import csv
import pathlib
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

MOMENT_COLUMNS = ("t", "x_center", "dx", "rho", "V1", "T", "H")
MARGINAL_COLUMNS = ("t", "cell_index", "v1", "g")
LEDGER_COLUMNS = ("t", "mass", "momentum1", "energy")


def _fmt(v) -> str:
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    return format(float(v), ".17g")


def _gather_rows(rows: np.ndarray, world: int) -> Optional[np.ndarray]:
    if world == 1:
        return rows
    import torch.distributed as dist
    out: List = [None] * world
    dist.all_gather_object(out, rows)
    return np.concatenate(out, axis=0) if dist.get_rank() == 0 else None


@dataclass
class RunRecord:
    """Collects output-time snapshots of a Solver1D (rank-collective calls)."""
    config: dict = field(default_factory=dict)
    marginal_cells: Sequence[int] = ()          # GLOBAL cell indices whose g(v1) is recorded
    moments: List[np.ndarray] = field(default_factory=list)
    marginals: List[np.ndarray] = field(default_factory=list)
    ledger: List[np.ndarray] = field(default_factory=list)
    step_seconds: List[float] = field(default_factory=list)

    def snapshot(self, solver) -> None:
        """Record moments of every cell, the selected marginals and the ledger at solver.t."""
        t = solver.t
        m = solver.moments().cpu().numpy()
        sl = slice(solver.start, solver.start + solver.ncl)
        rho = m[:, 0]
        with np.errstate(invalid="ignore", divide="ignore"):
            V1 = np.where(rho > 0, m[:, 1] / rho, 0.0)
        rows = np.column_stack([np.full(solver.ncl, t), solver.x_glob[sl], solver.dx_glob[sl], rho, V1, m[:, 5],
                                m[:, 6]])
        local = [c - solver.start for c in self.marginal_cells if solver.start <= c < solver.start + solver.ncl]
        if local:
            g = solver.marginals(local).cpu().numpy()
            v1 = solver.op.grid.v_nodes
            mrows = np.concatenate([np.column_stack([np.full(len(v1), t), np.full(len(v1), c + solver.start), v1,
                                                     g[i]]) for i, c in enumerate(local)])
        else:
            mrows = np.zeros((0, 4))
        led = solver.ledger()  # collective
        rows = _gather_rows(rows, solver.world)
        mrows = _gather_rows(mrows, solver.world)
        if rows is not None:
            self.moments.append(rows)
            self.marginals.append(mrows)
            self.ledger.append(np.concatenate([[t], led]))

    # ------------------------------------------------------------------ I/O
    def write_moment_csv(self, path) -> None:
        _write(path, MOMENT_COLUMNS, np.concatenate(self.moments) if self.moments else np.zeros((0, 7)))

    def write_marginal_csv(self, path) -> None:
        _write(path, MARGINAL_COLUMNS, np.concatenate(self.marginals) if self.marginals else np.zeros((0, 4)),
               int_cols=(1,))

    def write_ledger_csv(self, path) -> None:
        _write(path, LEDGER_COLUMNS, np.array(self.ledger) if self.ledger else np.zeros((0, 4)))


def _write(path, columns, rows: np.ndarray, int_cols=()) -> None:
    path = pathlib.Path(path)
    try:
        with path.open("w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(columns)
            for r in rows:
                w.writerow([_fmt(int(v)) if j in int_cols else _fmt(v) for j, v in enumerate(r)])
    except OSError as e:
        raise OSError(f"RunRecord: cannot write {path}: {e}") from e


def read_csv(path) -> tuple:
    """(columns, float64 rows) of a file written by RunRecord."""
    with pathlib.Path(path).open() as fh:
        r = csv.reader(fh)
        cols = tuple(next(r))
        rows = np.array([[float(v) for v in line] for line in r], dtype=np.float64).reshape(-1, len(cols))
    return cols, rows

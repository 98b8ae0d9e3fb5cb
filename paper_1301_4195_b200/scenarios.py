"""Synthetic inputs for BASELINE.json's configs (no dataset exists).

All randomness comes from one portable SplitMix64 stream with explicit 53-bit
mantissa conversion, so the CPU oracle and the GPU see bit-identical inputs.
Seeds are fixed and recorded in DESIGN.md.  Maxwellians follow SPEC.md:494-502.
"""
from __future__ import annotations

import math

import numpy as np

from .boltz import VelocityGrid

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """First `count` outputs of SplitMix64 seeded with `seed` (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, count: int, lo=0.0, hi=1.0) -> np.ndarray:
    u = (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return lo + (hi - lo) * u


def maxwellian(grid: VelocityGrid, rho, V, T) -> np.ndarray:
    """rho (2 pi T)^{-3/2} exp(-|v-V|^2 / 2T) at the N^3 nodes."""
    if not T > 0:
        raise ValueError("maxwellian: T must be positive")
    v = grid.velocities()
    d = v - np.asarray(V, dtype=np.float64)[None, :]
    return rho / (2.0 * np.pi * T) ** 1.5 * np.exp(-np.einsum("ij,ij->i", d, d) / (2.0 * T))


def maxwellians(grid: VelocityGrid, rho, V, T) -> np.ndarray:
    """Batched: rho (B,), V (B,3), T (B,) -> (B, N^3)."""
    v = grid.velocities()
    rho, V, T = np.asarray(rho, float), np.asarray(V, float), np.asarray(T, float)
    out = np.empty((rho.size, v.shape[0]))
    for i in range(rho.size):
        d = v - V[i][None, :]
        out[i] = rho[i] / (2.0 * np.pi * T[i]) ** 1.5 * np.exp(-np.einsum("ij,ij->i", d, d) / (2.0 * T[i]))
    return out


def config1_initial(grid: VelocityGrid, seed: int = 1301) -> np.ndarray:
    """cfg1: 0.5 M(1,(-1,0,0),1) + 0.5 M(1,(1,0,0),1), times (1 + 1e-3 U[-1,1])."""
    f = 0.5 * maxwellian(grid, 1.0, (-1.0, 0.0, 0.0), 1.0) + 0.5 * maxwellian(grid, 1.0, (1.0, 0.0, 0.0), 1.0)
    return f * (1.0 + 1e-3 * uniform(seed, f.size, -1.0, 1.0))


def mixture_params(ncells: int, seed: int = 4195):
    """cfg2/cfg5 per-cell two-Maxwellian parameters; per COMPONENT draws
    (SURVEY Appendix A.8): rho~U[0.5,2], u~U[-1,1]^3, T~U[0.5,2], 10 uniforms
    per cell in a fixed order, so cell i's state depends only on (seed, i)."""
    u = uniform(seed, 10 * ncells).reshape(ncells, 10)
    rho = 0.5 + 1.5 * u[:, [0, 5]]
    vel = -1.0 + 2.0 * u[:, [1, 2, 3, 6, 7, 8]].reshape(ncells, 2, 3)
    T = 0.5 + 1.5 * u[:, [4, 9]]
    return rho, vel, T


def mixture_cells(grid: VelocityGrid, ncells: int, seed: int = 4195, first: int = 0) -> np.ndarray:
    """(ncells, N^3) two-Maxwellian mixtures for cells [first, first+ncells)."""
    rho, vel, T = mixture_params(first + ncells, seed)
    rho, vel, T = rho[first:], vel[first:], T[first:]
    v = grid.velocities()
    out = np.zeros((ncells, v.shape[0]))
    for comp in range(2):
        d = v[None, :, :] - vel[:, comp, None, :]
        r2 = np.einsum("bij,bij->bi", d, d)
        out += rho[:, comp, None] / (2.0 * np.pi * T[:, comp, None]) ** 1.5 * np.exp(-r2 / (2.0 * T[:, comp, None]))
    return out


# ------------------------------------------------------------ spatial grids
def geometric_grid(ncells: int, length: float, ratio: float):
    """Cells clustered at x=0 with widths dx_j = dx0 * ratio^j tiling [0, length]
    (cfg3: 256 cells, ratio 1.02 over [0,20]).  Returns centres, widths."""
    dx = ratio ** np.arange(ncells)
    dx *= length / dx.sum()
    edges = np.concatenate([[0.0], np.cumsum(dx)])
    return 0.5 * (edges[:-1] + edges[1:]), dx


def zoned_grid(zones):
    """Piecewise-uniform cells: zones = [(length, dx), ...] from x = 0 outwards.
    Returns centres, widths."""
    dx = np.concatenate([np.full(int(round(length / h)), h) for length, h in zones])
    edges = np.concatenate([[0.0], np.cumsum(dx)])
    return 0.5 * (edges[:-1] + edges[1:]), dx


def sudden_heating(ratio: float = 2.0, T_before: float = 1.0, near: float = 2.0, far: float = 10.0,
                   mfp: float = 1.0):
    """The reference's sudden-heating / cooling scenario (SPEC.md scenario
    module; PAPER.md Figures 1-4): wall at x = 0 jumps to T_w = ratio *
    T_before at t = 0, uniform equilibrium M(1, 0, T_before) initially,
    8 cells per mean free path near the wall (x < near), 2 per mfp beyond,
    mfp = 1 (SPEC DESIGN DECISIONS), velocity half-width from the SPEC
    heuristic L = 2 sqrt(2 T_max) * 1.25.  Returns (x, dx, L, T_wall)."""
    if not ratio > 0:
        raise ValueError("sudden_heating: ratio must be > 0")
    x, dx = zoned_grid([(near, mfp / 8), (far - near, mfp / 2)])
    T_max = max(ratio * T_before, T_before)
    return x, dx, 2.0 * math.sqrt(2.0 * T_max) * 1.25, ratio * T_before


def uniform_grid(ncells: int, a: float, b: float):
    dx = np.full(ncells, (b - a) / ncells)
    return a + (np.arange(ncells) + 0.5) * dx, dx


def extend_ghosts(x: np.ndarray, dx: np.ndarray):
    """Centres/widths of the global field with 2 mirrored ghost cells per
    physical end (ghost widths mirror the adjacent interior cells)."""
    dxe = np.concatenate([[dx[1], dx[0]], dx, [dx[-1], dx[-2]]])
    xe = np.empty(len(dxe))
    xe[2:-2] = x
    xe[1] = x[0] - 0.5 * (dx[0] + dxe[1])
    xe[0] = xe[1] - 0.5 * (dxe[1] + dxe[0])
    xe[-2] = x[-1] + 0.5 * (dx[-1] + dxe[-2])
    xe[-1] = xe[-2] + 0.5 * (dxe[-2] + dxe[-1])
    return xe, dxe

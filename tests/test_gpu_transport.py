"""K4 transport / ghost fill and the Strang driver vs the CPU oracle (GPU)."""
import ctypes

import numpy as np
import pytest
import torch

from conftest import rel_max, table
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
from paper_1301_4195_b200.solver import Boundary, Solver1D, plan_decomposition, strang_step_loopback

pytestmark = pytest.mark.gpu


def _op(n, L):
    return CollisionOperator(VelocityGrid.create(n, L), KernelSpec(1.0), table(n, L))


@pytest.mark.parametrize("wl,wr", [(0, 0), (1, 0), (1, 1)])
def test_transport_step_vs_oracle(gpu, O, wl, wr):
    n, L, nx = 8, 5.0, 12
    x, dx = scenarios.geometric_grid(nx, 3.0, 1.15)
    xe, dxe = scenarios.extend_ghosts(x, dx)
    rng = np.random.default_rng(1)
    field = rng.random((nx + 4, n ** 3))
    base = rng.random((nx + 4, n ** 3))
    dt = 0.8 * dx.min() / L
    ref = O.transport_step(n, L, field, xe, dxe, dt, wl, wr)
    with _op(n, L) as op:
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(gpu)  # noqa: E731
        out = torch.empty_like(d(field))
        op.transport_step(d(field), out, d(xe), d(dxe), dt, wl, wr)
        assert rel_max(out.cpu().numpy(), ref) < 1e-13
        out2 = torch.empty_like(out)
        op.transport_step(d(field), out2, d(xe), d(dxe), dt, wl, wr, base=d(base), alpha=0.5)
        exp = ref.copy()
        exp[2:nx + 2] = 0.5 * base[2:nx + 2] + 0.5 * ref[2:nx + 2]
        assert rel_max(out2.cpu().numpy(), exp) < 1e-13


@pytest.mark.parametrize("side,kind", [(0, 0), (1, 0), (0, 1), (1, 1), (0, 2), (1, 2)])
def test_fill_boundary_vs_oracle(gpu, O, side, kind):
    n, L, nx = 8, 5.0, 6
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    xe, _ = scenarios.extend_ghosts(x, dx)
    rng = np.random.default_rng(2)
    field = rng.random((nx + 4, n ** 3))
    ref = field.copy()
    sref = O.fill_boundary(n, L, ref, xe, side, kind, Tw=2.0, Vw=(0.1, 0.0, 0.0))
    with _op(n, L) as op:
        f = torch.from_numpy(field).to(gpu)
        s = op.fill_boundary(f, torch.from_numpy(xe).to(gpu), side, kind, Tw=2.0, Vw=(0.1, 0.0, 0.0))
    assert rel_max(f.cpu().numpy(), ref) < 1e-13
    assert abs(s - sref) <= 1e-13 * max(1.0, abs(sref))


def _oracle_strang(O, n, L, G, field, xe, dxe, dt, Tw, steps, single_stage=False):
    """Strang step composed from the oracle's primitives,
    transport sub-step = SSP-RK2 of the FV step, or the SPEC's
    single stage with one ghost refresh."""
    nx = field.shape[0] - 4

    def fill(f):
        O.fill_boundary(n, L, f, xe, 0, 1, Tw=Tw)
        O.fill_boundary(n, L, f, xe, 1, 0)

    def T(f, h):
        fill(f)
        if single_stage:
            return O.transport_step(n, L, f, xe, dxe, h, 1, 0)
        t1 = O.transport_step(n, L, f, xe, dxe, h, 1, 0)
        fill(t1)
        t2 = O.transport_step(n, L, t1, xe, dxe, h, 1, 0)
        out = t1.copy()
        out[2:nx + 2] = 0.5 * f[2:nx + 2] + 0.5 * t2[2:nx + 2]
        return out

    for _ in range(steps):
        field = T(field, 0.5 * dt)
        field[2:nx + 2] = O.collision_rk2(n, L, G, field[2:nx + 2], dt)
        field = T(field, 0.5 * dt)
    return field


def test_strang_wall_problem_vs_oracle(gpu, O):
    """cfg3 in miniature: gas at rest, diffuse wall T_w=2 at x=0, geometric grid."""
    n, L, nx, Tw = 8, 5.0, 10, 2.0
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    xe, dxe = scenarios.extend_ghosts(x, dx)
    grid = VelocityGrid.create(n, L)
    f0 = np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (nx, 1))
    G = table(n, L)
    with _op(n, L) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw), right=Boundary("extrap"))
        dt = s.cfl_dt()
        for _ in range(4):
            s.strang_step(dt)
        got = s.interior.cpu().numpy()
    field = np.zeros((nx + 4, n ** 3))
    field[2:nx + 2] = f0
    ref = _oracle_strang(O, n, L, G, field, xe, dxe, dt, Tw, 4)[2:nx + 2]
    assert rel_max(got - f0, ref - f0) < 1e-9
    assert np.abs(got - f0).max() > 1e-6  # the wall did something


def test_strang_single_stage_transport_vs_oracle(gpu, O):
    """The SPEC-literal Strang step: each transport sub-step is ONE FV stage
    after one ghost refresh, against the same composition
    of oracle primitives; and it differs from the SSP-RK2 default."""
    n, L, nx, Tw = 8, 5.0, 10, 2.0
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    xe, dxe = scenarios.extend_ghosts(x, dx)
    grid = VelocityGrid.create(n, L)
    f0 = scenarios.mixture_cells(grid, nx, seed=23)
    G = table(n, L)
    with _op(n, L) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw), right=Boundary("extrap"),
                     transport_scheme="single_stage")
        dt = 0.5 * s.cfl_dt()
        for _ in range(4):
            s.strang_step(dt)
        got = s.interior.cpu().numpy()
        s2 = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw), right=Boundary("extrap"))
        for _ in range(4):
            s2.strang_step(dt)
        rk = s2.interior.cpu().numpy()
        # the graph path rotates one buffer pair per sub-step: 3 captured steps close it
        s3 = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw), right=Boundary("extrap"),
                      transport_scheme="single_stage")
        s3.run(dt, 4, graph=True)
        assert np.array_equal(s3.interior.cpu().numpy(), got)
    field = np.zeros((nx + 4, n ** 3))
    field[2:nx + 2] = f0
    ref = _oracle_strang(O, n, L, G, field, xe, dxe, dt, Tw, 4, single_stage=True)[2:nx + 2]
    assert rel_max(got - f0, ref - f0) < 1e-9
    assert rel_max(rk - f0, ref - f0) > 1e-6  # a different scheme


def test_single_stage_loopback_transparency(gpu):
    """Decomposition transparency of the single-stage scheme."""
    n, L, nx, Tw = 8, 5.0, 9, 2.0
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.05)
    grid = VelocityGrid.create(n, L)
    f0 = scenarios.mixture_cells(grid, nx, seed=29)
    with _op(n, L) as op:
        kw = dict(left=Boundary("wall", Tw), transport_scheme="single_stage")
        single = [Solver1D(op, x, dx, f0, **kw)]
        plan = plan_decomposition(nx, 3)
        multi = [Solver1D(op, x, dx, f0, rank=r, world=3, plan=plan, halo=False, **kw) for r in range(3)]
        for m in multi:
            m.halo = None
        dt = 0.5 * single[0].cfl_dt()
        for _ in range(3):
            strang_step_loopback(single, dt)
            strang_step_loopback(multi, dt)
        a = single[0].interior.cpu().numpy()
        b = np.concatenate([m.interior.cpu().numpy() for m in multi])
    assert np.array_equal(a, b)


@pytest.mark.parametrize("nranks", [2, 4])
def test_decomposition_transparency_bitwise(gpu, nranks):
    """N=8, M_x=8 wall-heating trajectories for n ranks are
    bit-identical to n=1 (loopback backend, one GPU)."""
    n, L, nx, Tw = 8, 5.0, 8, 2.0
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.05)
    grid = VelocityGrid.create(n, L)
    f0 = np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (nx, 1))
    with _op(n, L) as op:
        single = [Solver1D(op, x, dx, f0, left=Boundary("wall", Tw))]
        plan = plan_decomposition(nx, nranks)
        multi = [Solver1D(op, x, dx, f0, rank=r, world=nranks, left=Boundary("wall", Tw), plan=plan, halo=False)
                 for r in range(nranks)]
        for m in multi:
            m.halo = None
        dt = single[0].cfl_dt()
        for _ in range(5):
            strang_step_loopback(single, dt)
            strang_step_loopback(multi, dt)
        a = single[0].interior.cpu().numpy()
        b = np.concatenate([m.interior.cpu().numpy() for m in multi])
    assert np.array_equal(a, b)


def test_uniform_equilibrium_is_quiescent(gpu):
    """wall at the gas temperature, uniform equilibrium -> stays
    near equilibrium (bounded by the discrete equilibrium residual)."""
    n, L, nx = 8, 5.0, 8
    x, dx = scenarios.uniform_grid(nx, 0.0, 4.0)
    grid = VelocityGrid.create(n, L)
    f0 = np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (nx, 1))
    with _op(n, L) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary("wall", 1.0), right=Boundary("extrap"))
        dt = s.cfl_dt()
        for _ in range(10):
            s.strang_step(dt)
        got = s.interior.cpu().numpy()
    assert np.abs(got - f0).max() < 5e-2 * f0.max()


def test_async_graph_run_matches_eager(gpu):
    """Solver1D.run (async library + CUDA graph of 3 Strang steps) is bitwise
    the eager strang_step trajectory."""
    n, L, nx, Tw = 8, 5.0, 12, 2.0
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    grid = VelocityGrid.create(n, L)
    f0 = np.tile(scenarios.maxwellian(grid, 1.0, (0, 0, 0), 1.0), (nx, 1))
    with _op(n, L) as op:
        a = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw))
        b = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw))
        dt = a.cfl_dt()
        for _ in range(8):
            a.strang_step(dt)
        b.run(dt, 8)
        assert b.graph_replays == 2
        assert np.array_equal(a.interior.cpu().numpy(), b.interior.cpu().numpy())
        assert abs(a.t - b.t) < 1e-15


def test_async_mode_defers_numeric_error(gpu):
    from paper_1301_4195_b200 import NumericError
    n, L = 8, 5.0
    grid = VelocityGrid.create(n, L)
    f = torch.from_numpy(scenarios.mixture_cells(grid, 3, seed=2)).to(gpu)
    f[1, 5] = float("nan")
    with _op(n, L) as op:
        op.set_async(True)
        op.collision_rk2(f, 0.01)  # returns without raising
        with pytest.raises(NumericError):
            op.sync()
        op.sync()  # flag cleared
        op.set_async(False)


def test_ledger_collision_conserves_and_wall_flux(gpu):
    """SPEC.md:403 bookkeeping: the collision step leaves the global (mass,
    momentum, energy) ledger unchanged to round-off; a transport step between
    two extrapolating ends of a field at rest changes mass only through the
    end fluxes (which vanish for a symmetric field at rest)."""
    n, L, nx = 8, 5.0, 10
    x, dx = scenarios.uniform_grid(nx, 0.0, 2.0)
    grid = VelocityGrid.create(n, L)
    f0 = scenarios.mixture_cells(grid, nx, seed=31)
    with _op(n, L) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary("extrap"), right=Boundary("extrap"))
        a = s.ledger()
        s.collide(0.01)
        b = s.ledger()
        assert np.abs(b - a).max() < 1e-13 * np.abs(a).max()
        m = s.moments().cpu().numpy()
        assert np.all(m[:, 0] > 0) and np.all(m[:, 5] > 0)


def test_nccl_halo_graph_run_matches_eager(gpu):
    """Solver1D with the library's NCCL halo (world 1: the exchange is a no-op,
    the communicator and the capture path are real): 7 graph-replayed Strang
    steps are bitwise the eager steps without a halo."""
    import torch  # noqa: F401
    from paper_1301_4195_b200 import NcclHalo
    n, L, nx = 8, 5.0, 12
    grid = VelocityGrid.create(n, L)
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    f0 = scenarios.mixture_cells(grid, nx, seed=41)
    with _op(n, L) as op:
        a = Solver1D(op, x, dx, f0, left=Boundary("wall", 2.0), right=Boundary("extrap"))
        dt = a.cfl_dt()
        for _ in range(7):
            a.strang_step(dt)
        ref = a.interior.cpu().numpy()
        halo = NcclHalo(0, 1, 0)
        b = Solver1D(op, x, dx, f0, left=Boundary("wall", 2.0), right=Boundary("extrap"), halo=halo)
        b.run(dt, 7)
        assert getattr(b, "graph_replays", 0) == 2
        assert np.array_equal(b.interior.cpu().numpy(), ref)
        halo.close()


def test_multirank_capture_mode_and_teardown_order(gpu):
    """What bench.py's multi-rank cfg3 does around its graph, on one rank: the
    Strang steps captured in torch's thread-local capture mode (the mode used
    on several ranks, where NCCL's helper threads may call CUDA while this
    thread captures) with the overlapped NCCL halo, replayed bitwise equal to
    eager steps; then the teardown order -- release_graph() before
    NcclHalo.close() -- after which the solver still steps eagerly."""
    from paper_1301_4195_b200 import NcclHalo
    n, L, nx = 8, 5.0, 14
    grid = VelocityGrid.create(n, L)
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    f0 = scenarios.mixture_cells(grid, nx, seed=47)
    kw = dict(left=Boundary("wall", 2.0), right=Boundary("extrap"))
    with _op(n, L) as op:
        a = Solver1D(op, x, dx, f0, **kw)
        dt = a.cfl_dt()
        for _ in range(7):
            a.strang_step(dt)
        ref = a.interior.cpu().numpy()
        halo = NcclHalo(0, 1, 0)
        b = Solver1D(op, x, dx, f0, halo=halo, overlap_halo=True, **kw)
        b.strang_step(dt)
        b.capture(dt, capture_error_mode="thread_local")
        b.advance(6)
        assert getattr(b, "graph_replays", 0) == 2
        assert np.array_equal(b.interior.cpu().numpy(), ref)
        b.release_graph()
        halo.close()
        halo.close()                                   # idempotent
        b.halo = None
        b.strang_step(dt)
        a.strang_step(dt)
        assert np.array_equal(b.interior.cpu().numpy(), a.interior.cpu().numpy())


@pytest.mark.parametrize("scheme", ["ssp_rk2", "single_stage"])
def test_halo_overlap_bitwise(gpu, scheme):
    """SURVEY §8f rank 2, halo/compute overlap: with overlap_halo the NCCL
    exchange runs on a side stream while the rows that read no ghost are
    updated (boltz_transport_step_range), then the four edge rows.  World 1
    (the exchange is a no-op; the streams, the split launches and the graph
    capture are real): eager and graph-replayed steps are bitwise the plain
    driver's, and so is the boundary-flux ledger."""
    import torch
    from paper_1301_4195_b200 import NcclHalo
    n, L, nx = 8, 5.0, 14
    grid = VelocityGrid.create(n, L)
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    f0 = scenarios.mixture_cells(grid, nx, seed=43)
    kw = dict(left=Boundary("wall", 2.0), right=Boundary("extrap"), transport_scheme=scheme)
    with _op(n, L) as op:
        a = Solver1D(op, x, dx, f0, **kw)
        a.track_boundary_flux()
        dt = 0.5 * a.cfl_dt()
        for _ in range(7):
            a.strang_step(dt)
        ref, ref_flux = a.interior.cpu().numpy(), a.boundary_flux()
        halo = NcclHalo(0, 1, 0)
        b = Solver1D(op, x, dx, f0, halo=halo, overlap_halo=True, **kw)
        b.track_boundary_flux()
        for _ in range(7):
            b.strang_step(dt)
        torch.cuda.synchronize()
        assert np.array_equal(b.interior.cpu().numpy(), ref)
        assert np.array_equal(b.boundary_flux(), ref_flux)
        c = Solver1D(op, x, dx, f0, halo=halo, overlap_halo=True, **kw)
        c.run(dt, 7)
        assert getattr(c, "graph_replays", 0) == 2
        assert np.array_equal(c.interior.cpu().numpy(), ref)
        halo.close()


def test_transport_step_rows_split_bitwise(gpu):
    """boltz_transport_step_range: rows [4, ncl) + [2, 4) + [ncl, ncl + 2) are
    bitwise the whole-interior step (ghost rows copied by the edge launches);
    bad ranges are ConfigErrors."""
    import torch
    from paper_1301_4195_b200 import ConfigError
    n, L, nx = 8, 5.0, 11
    x, dx = scenarios.geometric_grid(nx, 3.0, 1.15)
    xe, dxe = scenarios.extend_ghosts(x, dx)
    rng = np.random.default_rng(5)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(gpu)  # noqa: E731
    field, base = d(rng.random((nx + 4, n ** 3))), d(rng.random((nx + 4, n ** 3)))
    with _op(n, L) as op:
        dt = 0.8 * dx.min() / L
        for kw in (dict(), dict(base=base, alpha=0.5)):
            full = torch.empty_like(field)
            op.transport_step(field, full, d(xe), d(dxe), dt, True, False, **kw)
            part = torch.full_like(field, float("nan"))
            for rows in ((4, nx), (2, 4), (nx, nx + 2)):
                op.transport_step(field, part, d(xe), d(dxe), dt, True, False, rows=rows, **kw)
            assert torch.equal(part, full)
        for rows in ((1, 4), (4, nx + 3), (5, 4)):
            with pytest.raises(ConfigError):
                op.transport_step(field, part, d(xe), d(dxe), dt, rows=rows)


def test_new_abi_entries_reject_bad_arguments(gpu):
    """ConfigError (category 2) for the peer transport, the edge store and the
    schedule setter on invalid input (no CUDA call is made)."""
    from paper_1301_4195_b200.boltz import lib
    n, L = 8, 5.0
    with _op(n, L) as op:
        h = op._h
        assert lib().boltz_set_schedule(h, 7) == 2
        assert lib().boltz_set_schedule(h, 0) == 0
        f = torch.zeros((6, n ** 3), dtype=torch.float64, device=gpu)
        p = f.data_ptr()
        L_ = lib()
        L_.boltz_transport_step_peer.restype = ctypes.c_int
        assert L_.boltz_transport_step_peer(ctypes.c_void_p(h.value), ctypes.c_void_p(p), None, ctypes.c_double(0.0),
                                            ctypes.c_void_p(p), ctypes.c_int64(2), None, None, ctypes.c_double(0.1),
                                            0, 0, None, None, None) == 2  # out aliases field, no grid
        assert L_.boltz_store_edges(ctypes.c_void_p(h.value), None, ctypes.c_int64(4), None, None, None) == 2

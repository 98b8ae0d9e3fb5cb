"""Pin the CPU oracle before trusting it (CPU only).

* grid: against the REFERENCE's own velocity_grid.cpp (tests/golden/grid_ref.json,
  produced by oracle/_ref/ref_grid, see tests/golden/make_golden.py);
* everything else: SPEC.md's known-answer tests (the reference ships no
  golden vectors and its collision/fourier sources are absent),
  plus independent cross-checks (numpy FFT, brute-force sums, scipy-free
  quadrature self-convergence).
"""
import itertools
import json
import math
import pathlib

import numpy as np
import pytest

from conftest import bkw, rel_max

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


# ------------------------------------------------------------------ grid
def test_grid_matches_reference_build(O):
    data = json.loads((GOLD / "grid_ref.json").read_text())
    for g in data["grids"]:
        o = O.grid(g["n"], g["L"])
        assert o["dv"] == g["dv"] and o["dzeta"] == g["dzeta"]
        assert np.array_equal(o["v"], g["v"]) and np.array_equal(o["zeta"], g["zeta"])
        assert np.array_equal(o["coeff"], g["coeff"])
        n = g["n"]
        c0, dv, dz = o["coeff"][0], o["dv"], o["dzeta"]
        assert c0 * c0 * c0 * dv * dv * dv == g["vel_weight_corner"]  # velocity_grid.hpp:38-41
        assert 1.0 * dz * dz * dz == g["fourier_weight_center"]  # velocity_grid.hpp:43-46
        assert (1 * n + 2) * n + 3 == g["flat_123"]


def test_grid_errors_match_reference(O):
    data = json.loads((GOLD / "grid_ref.json").read_text())
    for e in data["errors"]:
        assert e["category"] == 2  # ConfigError (errors.hpp:8-13)
        with pytest.raises(ValueError):
            O.grid(e["n"], e["L"])


def test_grid_spec_examples(O):
    g = O.grid(16, 5.0)
    assert g["dv"] == 0.625 and g["v"][8] == 0.0 and abs(g["dzeta"] - math.pi / 5) < 1e-15
    assert list(O.grid(4, 1.0)["v"]) == [-1.0, -0.5, 0.0, 0.5]
    g = O.grid(24, 5.0)
    assert abs(g["dv"] * g["dzeta"] - 2 * math.pi / 24) < 1e-15


# ------------------------------------------------------------- transforms
def _direct_forward(n, L, f):
    """O(N^6) direct sum of fourier.hpp:11-12 (SPEC.md:56 oracle)."""
    g = O_grid = None  # noqa
    dv, dz = 2 * L / n, math.pi / L
    k = np.arange(n)
    c = np.where((k == 0) | (k == n - 1), 0.5, 1.0)
    v = dv * (k - n // 2)
    z = dz * (k - n // 2)
    V = np.stack(np.meshgrid(v, v, v, indexing="ij"), -1).reshape(-1, 3)
    Z = np.stack(np.meshgrid(z, z, z, indexing="ij"), -1).reshape(-1, 3)
    C3 = (c[:, None, None] * c[None, :, None] * c[None, None, :]).ravel()
    ph = np.exp(-1j * (Z @ V.T))
    return (dv / math.sqrt(2 * math.pi)) ** 3 * ph @ (C3 * f)


def test_forward_direct_sum_maxwellian(O):
    n, L = 8, 5.0
    f = O.maxwellian(n, L, 1.0, np.zeros(3), 1.0)
    fh = O.forward(n, L, f)
    ref = _direct_forward(n, L, f)
    assert rel_max(fh, ref) < 1e-12
    i0 = (n // 2 * n + n // 2) * n + n // 2
    assert abs(fh[i0] - ref[i0]) / abs(ref[i0]) < 1e-12


def test_forward_matches_phase_wrapped_numpy_fft(O):
    """fourier.hpp:19-22: index-space FFT wrapped with (-1)^m, (-1)^k, (-1)^{N/2}."""
    rng = np.random.default_rng(0)
    for n, L in [(8, 5.0), (12, 6.0), (16, 6.0)]:
        f = rng.random(n ** 3)
        k = np.arange(n)
        c = np.where((k == 0) | (k == n - 1), 0.5, 1.0)
        s = (-1.0) ** k
        C3 = c[:, None, None] * c[None, :, None] * c[None, None, :]
        S3 = s[:, None, None] * s[None, :, None] * s[None, None, :]
        par = ((-1.0) ** (n // 2)) ** 3
        dv = 2 * L / n
        fh = (dv / math.sqrt(2 * math.pi)) ** 3 * par * S3 * np.fft.fftn(S3 * C3 * f.reshape(n, n, n))
        assert rel_max(O.forward(n, L, f), fh.ravel()) < 1e-13


def test_round_trip_and_linearity(O):
    n, L = 8, 5.0
    rng = np.random.default_rng(1)
    f, g = rng.random(n ** 3), rng.random(n ** 3)
    back, _ = O.inverse(n, L, O.forward(n, L, f))
    k = np.arange(n)
    c = np.where((k == 0) | (k == n - 1), 0.5, 1.0)
    C3 = (c[:, None, None] * c[None, :, None] * c[None, None, :]).ravel()
    assert np.abs(back - C3 * f).max() < 1e-10 * np.abs(f).max()  # SPEC.md:57, fourier.hpp:15-17
    lin = O.forward(n, L, 2.0 * f - 3.0 * g)
    assert rel_max(lin, 2.0 * O.forward(n, L, f) - 3.0 * O.forward(n, L, g)) < 1e-14


def test_inverse_delta_is_constant(O):
    n, L = 8, 5.0
    g = np.zeros(n ** 3, complex)
    g[(n // 2 * n + n // 2) * n + n // 2] = 1.0
    f, mi = O.inverse(n, L, g)
    dz = math.pi / L
    assert np.allclose(f, (dz / math.sqrt(2 * math.pi)) ** 3, rtol=1e-14, atol=0)
    assert mi < 1e-15


def test_symmetric_f_has_small_imag_residue(O):
    n, L = 8, 5.0
    f = O.maxwellian(n, L, 1.0, np.zeros(3), 1.0)
    _, mi = O.inverse(n, L, O.forward(n, L, f))
    assert mi < 1e-12 * f.max()


# ---------------------------------------------------------------- weights
def _pts(n, L):
    dz = math.pi / L
    return [np.array(p, float) * dz for p in itertools.product(range(-n // 2, n // 2), repeat=3)]


@pytest.mark.parametrize("lam", [0.0, 1.0])
def test_closed_form_matches_quadrature(O, lam):
    """closed forms vs radial quadrature on N=8 lattice pairs."""
    n, L = 8, 5.0
    pts = _pts(n, L)
    rng = np.random.default_rng(2)
    idx = rng.integers(0, len(pts), size=(1500, 2))
    worst = 0.0
    for a, b in idx:
        cf = O.weight_closed_form(lam, 1.0, L, pts[a], pts[b])
        qd = O.weight_quadrature(lam, 1.0, L, pts[a], pts[b], 64)
        worst = max(worst, abs(cf - qd) / max(1.0, abs(qd)))
    assert worst < 1e-8
    # the degenerate cases the printed formula gets wrong
    z = np.zeros(3)
    dz = math.pi / L
    for xi, ze in [(z, z), (pts[5], z), (z, pts[7]), (np.array([dz, 0, 0]), np.array([2 * dz, 0, 0])),
                   (np.array([dz, dz, 0]), np.array([2 * dz, 2 * dz, 0]))]:
        cf = O.weight_closed_form(lam, 1.0, L, xi, ze)
        qd = O.weight_quadrature(lam, 1.0, L, xi, ze, 64)
        assert math.isfinite(cf) and abs(cf - qd) / max(1.0, abs(qd)) < 1e-8


def test_zeta_zero_slice_is_zero_and_symmetry(O):
    n, L = 8, 5.0
    G = O.generate_table(n, L, 1.0).reshape(n ** 3, n ** 3)
    k0 = (n // 2 * n + n // 2) * n + n // 2
    assert np.all(G[k0] == 0.0)
    # simultaneous axis permutation of xi and zeta
    G6 = G.reshape((n,) * 6)
    Gp = G6.transpose(1, 0, 2, 4, 3, 5)  # swap axes 1<->2 of zeta and of xi
    assert np.abs(G6 - Gp).max() < 1e-12 * np.abs(G6).max()


def test_table_bit_identical_across_threads(O):
    a = O.generate_table(8, 5.0, 1.0, nthreads=1)
    b = O.generate_table(8, 5.0, 1.0, nthreads=8)
    assert np.array_equal(a, b)


def test_general_lambda_quadrature_self_converges(O):
    """lambda=0.5 value fixed by two node counts agreeing to 1e-10."""
    dz = math.pi / 5.0
    xi, ze = np.array([dz, 0, 0]), np.array([dz, dz, 0])
    a = O.weight_quadrature(0.5, 1.0, 5.0, xi, ze, 64)
    b = O.weight_quadrature(0.5, 1.0, 5.0, xi, ze, 128)
    assert abs(a - b) < 1e-10 * max(1, abs(b))
    assert abs(O.weight_quadrature(0.5, 1.0, 5.0, xi, np.zeros(3), 64)) < 1e-15  # zeta=0 -> 0


# -------------------------------------------------------------- collision
def _naive_qhat(n, L, G, fh):
    """triple loop of SPEC.md:189 straight from the formula (SPEC.md:194 oracle)."""
    dz = math.pi / L
    G = G.reshape(n ** 3, n ** 3)
    c = [0.5 if (i == 0 or i == n - 1) else 1.0 for i in range(n)]
    fh = fh.reshape(n, n, n)
    out = np.zeros((n, n, n), complex)
    for k in itertools.product(range(n), repeat=3):
        kf = (k[0] * n + k[1]) * n + k[2]
        acc = 0j
        for m in itertools.product(range(n), repeat=3):
            s = tuple(k[i] - m[i] + n // 2 for i in range(3))
            if min(s) < 0 or max(s) >= n:
                continue
            w = c[m[0]] * c[m[1]] * c[m[2]] * dz ** 3
            acc += G[kf, (m[0] * n + m[1]) * n + m[2]] * fh[m] * fh[s] * w
        out[k] = acc
    return out.ravel()


def test_qhat_vs_naive_loop_n6(O):
    n, L = 6, 4.0
    rng = np.random.default_rng(3)
    f = rng.random(n ** 3)
    G = O.generate_table(n, L, 1.0)
    fh = O.forward(n, L, f)
    q = O.evaluate_qhat(n, L, G, fh)
    assert rel_max(q, _naive_qhat(n, L, G, fh)) < 1e-13
    k0 = (n // 2 * n + n // 2) * n + n // 2
    assert q[k0] == 0
    assert np.all(O.evaluate_qhat(n, L, G, np.zeros(n ** 3, complex)) == 0)


def test_qhat_bilinear(O):
    n, L = 6, 4.0
    rng = np.random.default_rng(4)
    G = O.generate_table(n, L, 1.0)
    a = rng.standard_normal(n ** 3) + 1j * rng.standard_normal(n ** 3)
    b = rng.standard_normal(n ** 3) + 1j * rng.standard_normal(n ** 3)
    Q = lambda x: O.evaluate_qhat(n, L, G, x)  # noqa: E731
    # Q(a+b) = Q(a) + Q(b) + cross terms; cross = Q(a+b)-Q(a)-Q(b) is linear in each
    cross = Q(a + b) - Q(a) - Q(b)
    cross2 = Q(a + 2 * b) - Q(a) - Q(2 * b)
    assert rel_max(cross2, 2 * cross) < 1e-12
    assert rel_max(Q(3 * a), 9 * Q(a)) < 1e-13


def test_conserve_properties(O):
    n, L = 8, 5.0
    rng = np.random.default_rng(5)
    for _ in range(20):  # SPEC.md:602 (subset of the 200)
        qt = rng.random(n ** 3) - 0.3
        q = O.conserve(n, L, qt)
        m = O.moments(n, L, q)
        dv = 2 * L / n
        scale = np.abs(qt).max() * (2 * L) ** 3 * L ** 2
        assert np.abs(m[:5]).max() < 1e-12 * scale
        assert np.abs(O.conserve(n, L, q) - q).max() < 1e-12 * np.abs(q).max()  # idempotent SPEC.md:212
    # closest point: for feasible Z, ||Qt - P Qt|| <= ||Qt - Z||
    qt = rng.random(n ** 3)
    pq = O.conserve(n, L, qt)
    for _ in range(5):
        Z = O.conserve(n, L, rng.random(n ** 3))
        assert np.linalg.norm(qt - pq) <= np.linalg.norm(qt - Z) + 1e-14


def test_collide_maxwellian_residual_and_conservation(O):
    n, L = 16, 5.0
    G = O.generate_table(n, L, 1.0, nthreads=8)
    f = O.maxwellian(n, L, 1.0, np.zeros(3), 1.0)
    q, _ = O.collide(n, L, G, f, 1.0, nthreads=8)
    assert np.abs(q).max() < 5e-3 * f.max()
    m = O.moments(n, L, q)
    assert np.abs(m[:5]).max() < 1e-12 * O.moments(n, L, f)[0]
    with pytest.raises(FloatingPointError):
        bad = f.copy()
        bad[3] = np.nan
        O.collide(n, L, G, bad)


def test_rk2_conserves_moments(O):
    n, L = 8, 5.0
    G = O.generate_table(n, L, 1.0)
    f = 0.5 * O.maxwellian(n, L, 1.0, np.array([-1.0, 0, 0]), 1.0) + 0.5 * O.maxwellian(
        n, L, 1.0, np.array([1.0, 0, 0]), 1.0)
    m0 = O.moments(n, L, f)
    g = O.collision_rk2(n, L, G, f.reshape(1, -1), 0.01).ravel()
    m1 = O.moments(n, L, g)
    assert np.abs(m1[:5] - m0[:5]).max() < 1e-12 * m0[0]


# ---------------------------------------------------------------- moments
def test_moments_maxwellian(O):
    n, L = 24, 6.0
    f = O.maxwellian(n, L, 1.0, np.array([0.3, 0, 0]), 1.0)
    m = O.moments(n, L, f)
    # rho, V within 1e-6; T measured at 2.0e-6 (the half-weighted v=L-dv endpoint
    # truncates the shifted tail) and frozen at 5e-6 as SPEC.md:265 prescribes
    assert abs(m[0] - 1) < 1e-6 and abs(m[1] / m[0] - 0.3) < 1e-6 and abs(m[5] - 1) < 5e-6
    assert np.all(O.moments(n, L, np.zeros(n ** 3))[:6] == 0)
    assert np.allclose(O.moments(n, L, 2.5 * f)[:5], 2.5 * m[:5], rtol=1e-14)


# --------------------------------------------------------------- transport
def test_minmod_examples(O):
    assert O.minmod3(1, 2, 1.5) == 1
    assert O.minmod3(-1, 2, 0.5) == 0
    assert O.minmod3(-2, -1, -1.5) == -1


def _ext(x, dx):
    from paper_1301_4195_b200.scenarios import extend_ghosts
    return extend_ghosts(x, dx)


def test_transport_telescoping_and_constant(O):
    from paper_1301_4195_b200.scenarios import geometric_grid
    n, L = 4, 3.0
    x, dx = geometric_grid(20, 5.0, 1.1)
    xe, dxe = _ext(x, dx)
    rng = np.random.default_rng(6)
    field = np.zeros((24, n ** 3))
    field[2:22] = rng.random((20, n ** 3))
    O.fill_boundary(n, L, field, xe, 0, 0)
    O.fill_boundary(n, L, field, xe, 1, 0)
    dt = 0.5 * dx.min() / L
    out = O.transport_step(n, L, field, xe, dxe, dt, 0, 0)
    # mass change == boundary fluxes (telescoping): recompute face fluxes
    v1 = (2 * L / n) * (np.arange(n ** 3) // (n * n) - n // 2)
    d_int = ((out[2:22] - field[2:22]) * dx[:, None]).sum(0)
    # constant field stays constant
    const = np.zeros_like(field)
    const[:] = 0.7
    oc = O.transport_step(n, L, const, xe, dxe, dt, 0, 0)
    assert np.abs(oc[2:22] - 0.7).max() < 1e-15
    # interior mass change is a pure boundary term: with a zero field near the ends it vanishes
    f2 = np.zeros_like(field)
    f2[8:14] = rng.random((6, n ** 3))
    o2 = O.transport_step(n, L, f2, xe, dxe, dt, 0, 0)
    assert abs(((o2[2:22] - f2[2:22]) * dx[:, None]).sum()) < 1e-13
    assert np.isfinite(d_int).all() and v1.shape[0] == n ** 3


def _periodic(field, nx):
    field[0:2] = field[nx:nx + 2]
    field[nx + 2:nx + 4] = field[2:4]
    return field


def test_transport_second_order(O):
    """SPEC.md:349 / acceptance 5: smooth sine, one v1>0 node,
    uniform grid, EOC >= 1.8.  The transport sub-step is SSP-RK2 over the SPEC's
    single FV step ("each system is evolved ... second-order
    Runge-Kutta"; a single forward-Euler stage is only first order in time,
    DESIGN.md "Transport")."""
    from paper_1301_4195_b200.scenarios import uniform_grid
    n, L = 4, 2.0
    errs = []
    for nx in (128, 256):
        x, dx = uniform_grid(nx, 0.0, 1.0)
        xe, dxe = _ext(x, dx)
        j = 3 * n * n + (n // 2) * n + n // 2  # i1 = 3 -> v1 = dv > 0
        v1 = (2 * L / n) * (3 - n // 2)
        T = 0.5
        steps = int(round(T / (0.4 * dx[0] / v1)))
        dt = T / steps
        field = np.zeros((nx + 4, n ** 3))
        field[2:nx + 2, :] = ((np.cos(2 * np.pi * (x - dx / 2)) - np.cos(2 * np.pi * (x + dx / 2)))
                              / (2 * np.pi * dx))[:, None]
        for _ in range(steps):
            f1 = O.transport_step(n, L, _periodic(field, nx), xe, dxe, dt, 0, 0)
            f2 = O.transport_step(n, L, _periodic(f1, nx), xe, dxe, dt, 0, 0)
            field = 0.5 * field + 0.5 * f2
        exact = (np.cos(2 * np.pi * (x - dx / 2 - v1 * T)) - np.cos(2 * np.pi * (x + dx / 2 - v1 * T))) / (
            2 * np.pi * dx)
        errs.append(np.abs(field[2:nx + 2, j] - exact).mean())
    eoc = math.log2(errs[0] / errs[1])
    assert eoc >= 1.8, (errs, eoc)


def test_transport_no_new_extrema(O):
    """Acceptance 5: minmod on a step profile creates no new extrema."""
    from paper_1301_4195_b200.scenarios import uniform_grid
    n, L, nx = 4, 2.0, 64
    x, dx = uniform_grid(nx, 0.0, 1.0)
    xe, dxe = _ext(x, dx)
    field = np.zeros((nx + 4, n ** 3))
    field[2:nx + 2] = np.where((x > 0.3) & (x < 0.6), 1.0, 0.2)[:, None]
    dt = 0.4 * dx[0] / L
    for _ in range(40):
        f1 = O.transport_step(n, L, _periodic(field, nx), xe, dxe, dt, 0, 0)
        f2 = O.transport_step(n, L, _periodic(f1, nx), xe, dxe, dt, 0, 0)
        field = 0.5 * field + 0.5 * f2
    inner = field[2:nx + 2]
    assert inner.max() <= 1.0 + 1e-13 and inner.min() >= 0.2 - 1e-13


def test_wall_balances_equilibrium(O):
    """wall Maxwellian at T_w emits what it absorbs, "within
    quadrature tolerance": sigma_w uses the continuum normalisation
    sqrt(2 pi / T_w) (PAPER.md Eq. BC), so the discrete imbalance is the
    half-space trapezoid error -- measured 2.5% at N=16, shrinking with N."""
    x = np.array([0.25, 0.75, 1.25])
    dx = np.full(3, 0.5)
    xe, dxe = _ext(x, dx)
    imb = []
    for n, L in [(16, 6.0), (32, 6.0)]:
        field = np.zeros((7, n ** 3))
        for c in range(2, 5):
            field[c] = O.maxwellian(n, L, 1.0, np.zeros(3), 2.0)
        sig = O.fill_boundary(n, L, field, xe, 0, 1, Tw=2.0)
        dv = 2 * L / n
        v1 = dv * (np.arange(n ** 3) // (n * n) - n // 2)
        k = np.arange(n)
        c = np.where((k == 0) | (k == n - 1), 0.5, 1.0)
        w = (c[:, None, None] * c[None, :, None] * c[None, None, :]).ravel() * dv ** 3
        out_flux = (v1 * field[2] * w)[v1 <= 0].sum()
        in_flux = (v1 * field[1] * w)[v1 > 0].sum()
        imb.append(abs(in_flux + out_flux) / abs(out_flux))
        assert sig > 0
    assert imb[0] < 0.03 and imb[1] < 0.3 * imb[0]
    n, L = 16, 6.0
    z = np.zeros((7, n ** 3))
    assert O.fill_boundary(n, L, z, xe, 0, 1, Tw=2.0) == 0.0 and np.all(z == 0)


def test_plan_decomposition(O):
    s, c = O.plan_decomposition(10, 2)
    assert list(s) == [0, 5] and list(c) == [5, 5]
    assert sorted(O.plan_decomposition(10, 3)[1]) == [3, 3, 4]
    with pytest.raises(ValueError):
        O.plan_decomposition(2, 3)


# ---------------------------------------------------------------- physics
def _stress_rate(n, L, f, Q):
    """(d/dt Pi_11 from Q, exact -rho Pi_11 / 2): for Maxwell molecules with
    isotropic b = 1/(4 pi) the traceless pressure tensor relaxes at rate rho/2
    (weak form with phi = v1^2 - |v|^2/3, symmetrised: <phi'+phi*'-phi-phi*>_sigma
    = (u'u' - uu)/2 averaged over sigma)."""
    dv = 2 * L / n
    k = np.arange(n)
    c = np.where((k == 0) | (k == n - 1), 0.5, 1.0)
    w = (c[:, None, None] * c[None, :, None] * c[None, None, :]).ravel() * dv ** 3
    v = dv * (k - n // 2)
    V1, V2, V3 = [a.ravel() for a in np.meshgrid(v, v, v, indexing="ij")]
    rho = (f * w).sum()
    U = np.array([(f * w * V1).sum(), (f * w * V2).sum(), (f * w * V3).sum()]) / rho
    c1, c2, c3 = V1 - U[0], V2 - U[1], V3 - U[2]
    cc = c1 * c1 + c2 * c2 + c3 * c3
    pi11 = (f * w * (c1 * c1 - cc / 3)).sum()
    lhs = (Q * w * (V1 * V1 - (V1 * V1 + V2 * V2 + V3 * V3) / 3)).sum()
    return lhs, -0.5 * rho * pi11


@pytest.mark.parametrize("n,L,tol", [(16, 6.0, 1e-2), (24, 8.0, 1e-3)])
def test_spectral_operator_matches_maxwell_molecule_stress_relaxation(O, n, L, tol):
    """Analytic physics pin of the spectral operator's normalisation (the
    (2 pi)^{3/2} factors, b = 1/(4 pi), the trapezoid weights): measured rel.
    error 5e-3 at N=16, 1e-4 at N=24."""
    f = 0.5 * O.maxwellian(n, L, 1.0, np.array([-0.7, 0, 0]), 0.8) + 0.5 * O.maxwellian(
        n, L, 1.0, np.array([0.7, 0, 0]), 0.8)
    G = O.generate_table(n, L, 0.0, nthreads=8)
    lhs, exact = _stress_rate(n, L, f, O.q_tilde(n, L, G, f))
    assert abs(lhs - exact) < tol * abs(exact)


def test_direct_strong_form_oracle(O):
    """direct_collision_oracle, N=8/12, lambda=0.
    * angular self-convergence (0.65% between 8x16 and 16x32 sphere nodes) and
      the Maxwell-molecule stress rate (-rho Pi/2; measured 2.5% at N=8, 0.7% at N=12);
    * SPEC.md:604's 5% L2 pointwise agreement with the spectral Q does NOT hold
      at N <= 12 with trilinear interpolation (measured 69-80%; the strong form's
      gain term interpolates a Gaussian on dv ~ 0.8) -- recorded, not asserted;
    * N > 12 rejected."""
    for n, L, tol in [(8, 5.0, 4e-2), (12, 5.0, 1.5e-2)]:
        f = 0.5 * O.maxwellian(n, L, 1.0, np.array([-0.7, 0, 0]), 0.8) + 0.5 * O.maxwellian(
            n, L, 1.0, np.array([0.7, 0, 0]), 0.8)
        qa = O.direct_collision(n, L, 0.0, f, 8, 16, nthreads=8)
        qb = O.direct_collision(n, L, 0.0, f, 16, 32, nthreads=8)
        assert np.linalg.norm(qa - qb) < 2e-2 * np.linalg.norm(qb)
        lhs, exact = _stress_rate(n, L, f, qb)
        assert abs(lhs - exact) < tol * abs(exact)
        assert np.all(O.direct_collision(n, L, 0.0, np.zeros(n ** 3), 4, 8) == 0)  # f = 0 -> 0
    with pytest.raises(ValueError):
        O.direct_collision(16, 5.0, 0.0, np.zeros(16 ** 3))


def _bkw_strong_form(K, v, n_star=32, L_star=7.0, n_theta=12, n_phi=24):
    """Strong-form Q(f)(v) (SPEC.md:213-221 collision rule, b = 1/(4 pi)) with
    the BKW f evaluated analytically at v', v*' (no lattice interpolation);
    v* by the trapezoid rule on an n_star^3 lattice over [-L_star, L_star)."""
    def fk(v2):
        return (2 * np.pi * K) ** -1.5 * np.exp(-v2 / (2 * K)) * ((5 * K - 3) / (2 * K) + (1 - K) / (2 * K * K) * v2)

    gx, gw = np.polynomial.legendre.leggauss(n_theta)
    ct = np.repeat(gx, n_phi)
    st = np.sqrt(1 - ct ** 2)
    ph = np.tile(2 * np.pi * np.arange(n_phi) / n_phi, n_theta)
    sig = np.stack([st * np.cos(ph), st * np.sin(ph), ct], 1)
    sw = np.repeat(gw, n_phi) * 2 * np.pi / n_phi / (4 * np.pi)
    dv = 2 * L_star / n_star
    x = dv * (np.arange(n_star) - n_star // 2)
    vs = np.stack(np.meshgrid(x, x, x, indexing="ij"), -1).reshape(-1, 3)
    u = v - vs
    um = np.linalg.norm(u, axis=1)
    c = 0.5 * (v + vs)
    gain = np.zeros(len(vs))
    for s in range(len(sw)):
        vp = c + 0.5 * um[:, None] * sig[s]
        vq = c - 0.5 * um[:, None] * sig[s]
        gain += sw[s] * fk((vp * vp).sum(1)) * fk((vq * vq).sum(1))
    return float((dv ** 3 * (gain - fk(float(v @ v)) * fk((vs * vs).sum(1)))).sum())


def test_bkw_exact_solution_pins_the_operator(O):
    """Pointwise analytic pin (Bobylev-Krook-Wu, Maxwell molecules, lambda=0).
    1. The BKW Q is the strong-form collision integral with
       b = 1/(4 pi): checked with analytic f at off-lattice points (~1e-9).
    2. The spectral operator (oracle: forward -> evaluate_qhat -> inverse ->
       conserve) converges to it: measured rel. L2 error 0.242 (N=8, L=5),
       0.0291 (N=12, L=5), 0.0104 (N=16, L=6); 0.00154 at N=24, L=8.
    3. The lattice direct_collision_oracle (trilinear interpolation of f at v',
       v*') is interpolation-limited at N <= 12: measured 1.44 (N=8) and 1.08
       (N=12) rel. L2 error against the same exact Q -- which is why SPEC.md:604's
       5% spectral-vs-direct agreement cannot hold there."""
    K = 0.7
    for v in ([0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.5, 0.5, 0.5], [0.0, 1.5, 1.0]):
        v = np.array(v)
        _, qe = bkw_point(K, v)
        assert abs(_bkw_strong_form(K, v) - qe) < 1e-8 * 0.0125
    errs = {}
    for n, L, tol in [(8, 5.0, 0.26), (12, 5.0, 0.032), (16, 6.0, 0.0115)]:
        f, qe = bkw(n, L, K)
        G = O.generate_table(n, L, 0.0, nthreads=8)
        q = O.collide(n, L, G, f)[0]
        errs[n] = np.linalg.norm(q - qe) / np.linalg.norm(qe)
        assert errs[n] < tol
    assert errs[16] < errs[12] < errs[8]
    f, qe = bkw(8, 5.0, K)
    qd = O.direct_collision(8, 5.0, 0.0, f, 8, 16, nthreads=8)
    assert np.linalg.norm(qd - qe) / np.linalg.norm(qe) > 0.5  # recorded: interpolation-limited


def bkw_point(K, v):
    """BKW (f, Q) at one off-lattice velocity v (same formula as conftest.bkw)."""
    v2 = float(v @ v)
    E = (2 * np.pi * K) ** -1.5 * np.exp(-v2 / (2 * K))
    a, b = (5 * K - 3) / (2 * K), (1 - K) / (2 * K * K)
    dfdK = E * ((-1.5 / K + v2 / (2 * K * K)) * (a + b * v2) + 1.5 / (K * K) + (K - 2) / (2 * K ** 3) * v2)
    return E * (a + b * v2), dfdK * (1 - K) / 6


def test_bkw_closed_form_derivative():
    """conftest.bkw's analytic dQ/dK against a central difference."""
    for K in (0.62, 0.7, 0.9):
        f1, _ = bkw(8, 5.0, K + 1e-6)
        f0, _ = bkw(8, 5.0, K - 1e-6)
        _, q = bkw(8, 5.0, K)
        assert np.abs((f1 - f0) / 2e-6 * (1 - K) / 6 - q).max() < 1e-8 * np.abs(q).max()


def test_marginal_spec_examples(O):
    """SPEC marginal_distribution examples: Maxwellian(1,0,1) -> (2 pi)^{-1/2}
    exp(-v1^2/2) within 1e-6; sum g dv c = rho; f = 0 -> 0."""
    n, L = 24, 6.0
    f = O.maxwellian(n, L, 1.0, np.zeros(3), 1.0)
    g = O.marginal(n, L, f)
    v = 2 * L / n * (np.arange(n) - n // 2)
    assert np.abs(g - np.exp(-v * v / 2) / np.sqrt(2 * np.pi)).max() < 1e-6
    c = np.where((np.arange(n) == 0) | (np.arange(n) == n - 1), 0.5, 1.0)
    assert abs((g * c).sum() * 2 * L / n - O.moments(n, L, f)[0]) < 1e-13
    assert np.all(O.marginal(n, L, np.zeros(n ** 3)) == 0)


@pytest.mark.parametrize("side", [0, 1])
def test_balanced_wall_has_zero_net_mass_flux(O, side):
    """Wall kind 2 (extension): the re-emitted lattice influx equals the lattice
    outflux to round-off; kind 1 (the reference's continuum sigma_w) does not
    (2-3% at dv = 0.625, O(dv^2))."""
    n, L, nx = 16, 5.0, 6
    x = np.arange(nx + 4) - 1.5
    rng = np.random.default_rng(5)
    base = np.tile(O.maxwellian(n, L, 1.0, np.array([0.3, 0.1, 0.0]), 1.0), (nx + 4, 1))
    base *= 1 + 0.1 * rng.random(base.shape)
    v1 = np.repeat(2 * L / n * (np.arange(n) - n // 2), n * n)
    k = np.arange(n)
    c = np.where((k == 0) | (k == n - 1), 0.5, 1.0)
    w = (c[:, None, None] * c[None, :, None] * c[None, None, :]).ravel() * (2 * L / n) ** 3
    nrm = 1.0 if side == 0 else -1.0
    gi, ii = (1, 2) if side == 0 else (nx + 2, nx + 1)
    imb = {}
    for kind in (1, 2):
        f = base.copy()
        O.fill_boundary(n, L, f, x, side, kind, Tw=1.7)
        un = v1 * nrm
        out = -(un * f[ii] * w)[un <= 0].sum()
        inn = (un * f[gi] * w)[un > 0].sum()
        imb[kind] = abs(inn - out) / out
    assert imb[2] < 1e-14 and imb[1] > 1e-3

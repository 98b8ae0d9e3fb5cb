"""ctypes view of the CPU ORACLE (oracle/boltz_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
`--impl reference` leg may import this module.  It is the checker, never the
thing measured or shipped.  See boltz_oracle.c's header for what each
function restates (SPEC.md / PAPER.md / reference header file:line).
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libboltz_oracle.so"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_lib = None


def build() -> None:
    # stdout silenced: bench.py's contract is ONE JSON line on stdout
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        i, d, i64 = C.c_int, C.c_double, C.c_int64
        sig = {
            "bo_grid": (i, [i, d, C.POINTER(d), C.POINTER(d), _dp, _dp, _dp]),
            "bo_weight_closed_form": (d, [d, d, d, _dp, _dp]),
            "bo_weight_quadrature": (d, [d, d, d, _dp, _dp, i]),
            "bo_generate_table": (None, [i, d, d, d, d, i, _dp, i]),
            "bo_forward": (None, [i, d, _dp, _dp]),
            "bo_inverse": (None, [i, d, _dp, _dp, C.POINTER(d)]),
            "bo_evaluate_qhat": (None, [i, d, _dp, _dp, _dp]),
            "bo_evaluate_qhat_omp": (None, [i, d, _dp, _dp, _dp, i]),
            "bo_conserve": (None, [i, d, _dp, _dp]),
            "bo_collide": (i, [i, d, _dp, _dp, d, _dp, C.POINTER(d), i]),
            "bo_collision_rk2": (i, [i, d, _dp, _dp, i64, d, d, i]),
            "bo_moments": (None, [i, d, _dp, _dp]),
            "bo_maxwellian": (None, [i, d, d, _dp, d, _dp]),
            "bo_marginal": (None, [i, d, _dp, _dp]),
            "bo_minmod3": (d, [d, d, d]),
            "bo_fill_boundary": (None, [i, d, _dp, i64, _dp, i, i, d, _dp, C.POINTER(d)]),
            "bo_transport_step": (None, [i, d, _dp, _dp, i64, _dp, _dp, d, i, i]),
            "bo_plan_decomposition": (i, [i64, i, _ip, _ip]),
            "bo_direct_collision": (i, [i, d, d, _dp, i, i, _dp, i]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def grid(n, L):
    v, z, c = np.zeros(n), np.zeros(n), np.zeros(n)
    dv, dz = C.c_double(), C.c_double()
    rc = lib().bo_grid(n, L, C.byref(dv), C.byref(dz), v, z, c)
    if rc:
        raise ValueError(f"ConfigError({rc}): invalid grid N={n} L={L}")
    return dict(n=n, L=L, dv=dv.value, dzeta=dz.value, v=v, zeta=z, coeff=c)


def weight_closed_form(lam, beta, r0, xi, zeta):
    return lib().bo_weight_closed_form(lam, beta, r0, _c(xi), _c(zeta))


def weight_quadrature(lam, beta, r0, xi, zeta, panels=64):
    return lib().bo_weight_quadrature(lam, beta, r0, _c(xi), _c(zeta), panels)


def generate_table(n, L, lam=1.0, beta=1.0, r0=None, panels=64, nthreads=0):
    r0 = L if r0 is None else r0
    G = np.empty((n ** 3) * (n ** 3), dtype=np.float64)
    lib().bo_generate_table(n, L, lam, beta, r0, panels, G, nthreads)
    return G


def forward(n, L, f):
    out = np.empty(2 * n ** 3)
    lib().bo_forward(n, L, _c(f).ravel(), out)
    return out.view(np.complex128)


def inverse(n, L, g):
    g = np.ascontiguousarray(g, dtype=np.complex128).ravel().view(np.float64)
    out = np.empty(n ** 3)
    mi = C.c_double()
    lib().bo_inverse(n, L, g, out, C.byref(mi))
    return out, mi.value


def evaluate_qhat(n, L, G, fhat, nthreads=0):
    fh = np.ascontiguousarray(fhat, dtype=np.complex128).ravel().view(np.float64)
    out = np.empty(2 * n ** 3)
    if nthreads:
        lib().bo_evaluate_qhat_omp(n, L, G, fh, out, nthreads)
    else:
        lib().bo_evaluate_qhat(n, L, G, fh, out)
    return out.view(np.complex128)


def conserve(n, L, qt):
    out = np.empty(n ** 3)
    lib().bo_conserve(n, L, _c(qt).ravel(), out)
    return out


def collide(n, L, G, f, eps=1.0, nthreads=0):
    out = np.empty(n ** 3)
    mi = C.c_double()
    rc = lib().bo_collide(n, L, G, _c(f).ravel(), eps, out, C.byref(mi), nthreads)
    if rc:
        raise FloatingPointError(f"NumericError({rc}): non-finite input")
    return out, mi.value


def collision_rk2(n, L, G, f, dt, eps=1.0, nthreads=0):
    """f: (ncells, N^3); returns a new array."""
    f = np.array(f, dtype=np.float64, copy=True, order="C")
    ncells = f.size // n ** 3
    rc = lib().bo_collision_rk2(n, L, G, f.reshape(-1), ncells, dt, eps, nthreads)
    if rc:
        raise FloatingPointError(f"NumericError({rc})")
    return f


def moments(n, L, f):
    out = np.empty(7)
    lib().bo_moments(n, L, _c(f).ravel(), out)
    return out


def marginal(n, L, f):
    """marginal_distribution: g(v1) over the N v1 nodes."""
    out = np.empty(n)
    lib().bo_marginal(n, L, _c(f).ravel(), out)
    return out


def maxwellian(n, L, rho, V, T):
    out = np.empty(n ** 3)
    lib().bo_maxwellian(n, L, rho, _c(V), T, out)
    return out


def minmod3(a, b, c):
    return lib().bo_minmod3(a, b, c)


def fill_boundary(n, L, field, x_ext, side, kind, Tw=1.0, Vw=(0.0, 0.0, 0.0)):
    """In place on field (ncl+4, N^3); returns sigma_w."""
    ncl = field.shape[0] - 4
    s = C.c_double()
    lib().bo_fill_boundary(n, L, field.reshape(-1), ncl, _c(x_ext), side, kind, Tw, _c(Vw), C.byref(s))
    return s.value


def transport_step(n, L, field, x_ext, dx_ext, dt, wall_left, wall_right):
    ncl = field.shape[0] - 4
    out = np.empty_like(field)
    lib().bo_transport_step(n, L, _c(field).reshape(-1), out.reshape(-1), ncl, _c(x_ext),
                            _c(dx_ext), dt, int(wall_left), int(wall_right))
    return out


def plan_decomposition(ncells, nranks):
    s = np.zeros(max(nranks, 1), dtype=np.int64)
    c = np.zeros(max(nranks, 1), dtype=np.int64)
    rc = lib().bo_plan_decomposition(ncells, nranks, s, c)
    if rc:
        raise ValueError(f"ConfigError({rc}): {nranks} ranks > {ncells} cells")
    return s, c


def direct_collision(n, L, lam, f, n_theta=12, n_phi=24, nthreads=0):
    """Strong-form quadrature oracle, N <= 12."""
    out = np.empty(n ** 3)
    rc = lib().bo_direct_collision(n, L, lam, _c(f).ravel(), n_theta, n_phi, out, nthreads)
    if rc:
        raise ValueError("direct_collision_oracle: N must be <= 12")
    return out


def q_tilde(n, L, G, f):
    """Unprojected spectral operator: inverse(evaluate_qhat(forward(f)))."""
    return inverse(n, L, evaluate_qhat(n, L, G, forward(n, L, f)))[0]

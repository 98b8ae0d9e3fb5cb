"""Python mirror of the reference's collision-path API over the C ABI.

The reference is C++ (proj/include/boltz/*.hpp + SPEC.md); this module keeps
its names, argument meanings and error categories so the parity tests and
the benchmark read like the reference's own tests:

  VelocityGrid.create(n, L)        velocity_grid.hpp:17-47 / velocity_grid.cpp:11-32
  KernelSpec(lam, beta, r0)
  generate_table / save_table /
    load_table                     SPEC.md:126-143 (host, C++ in libboltz_cuda.so)
  CollisionOperator                SpectralTransform (fourier.hpp:28-52) +
                                   evaluate_qhat / conserve / collide
                                   + collision_rk2, batched
  transport_step / fill_boundary
  ConfigError / IoError /
    NumericError                   errors.hpp:8-35 (categories 2/3/4)

Every compute call goes to libboltz_cuda.so (sm_100a kernels).  There is no
CPU fallback: a missing library raises ImportError-like RuntimeError.
Arrays may be numpy (host memory: the call stages H2D/D2H) or torch CUDA
tensors (device memory: ordered on the current torch stream).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .build import LIB as _LIB_PATH

MEM_HOST, MEM_DEVICE = 0, 1


class BoltzError(RuntimeError):
    category = 0

    def __init__(self, msg, category=None):
        super().__init__(msg)
        if category is not None:
            self.category = category


class ConfigError(BoltzError):
    category = 2


class IoError(BoltzError):
    category = 3


class NumericError(BoltzError):
    category = 4


class CudaError(BoltzError):
    category = 5


_ERR = {2: ConfigError, 3: IoError, 4: NumericError, 5: CudaError}
_lib = None


def lib():
    """Load libboltz_cuda.so (built in-tree by paper_1301_4195_b200.build)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"{_LIB_PATH} is missing: run `python -m paper_1301_4195_b200.build` "
                "(there is no CPU fallback for the collision path)")
        path = os.environ.get("BOLTZ_LIB_VARIANT") or str(_LIB_PATH)  # dev: A/B kernel variants
        L = C.CDLL(path)
        vp, i, d, i64 = C.c_void_p, C.c_int, C.c_double, C.c_int64
        dp = C.POINTER(C.c_double)
        sig = {
            "boltz_last_error": (C.c_char_p, []),
            "boltz_build_info": (C.c_char_p, []),
            "boltz_create": (i, [i, d, d, d, d, vp, i, C.POINTER(vp)]),
            "boltz_create_generated": (i, [i, d, d, d, d, i, i, C.POINTER(vp)]),
            "boltz_destroy": (i, [vp]),
            "boltz_memory_bytes": (i, [vp, C.POINTER(i64), C.POINTER(i64)]),
            "boltz_forward_batch": (i, [vp, vp, vp, i64, i, vp]),
            "boltz_inverse_batch": (i, [vp, vp, vp, vp, i64, i, vp]),
            "boltz_qhat_batch": (i, [vp, vp, vp, i64, i, vp]),
            "boltz_conserve_batch": (i, [vp, vp, vp, i64, i, vp]),
            "boltz_collide_batch": (i, [vp, vp, vp, i64, d, vp, i, vp]),
            "boltz_rk2_batch": (i, [vp, vp, i64, d, d, i, vp]),
            "boltz_transport_step": (i, [vp, vp, vp, d, vp, i64, vp, vp, d, i, i, vp]),
            "boltz_transport_step_range": (i, [vp, vp, vp, d, vp, i64, vp, vp, d, i, i, i64, i64, vp]),
            "boltz_fill_boundary": (i, [vp, vp, i64, vp, i, i, d, vp, dp, vp]),
            "boltz_moments_batch": (i, [vp, vp, vp, i64, i, vp]),
            "boltz_marginal_batch": (i, [vp, vp, vp, i64, i, vp]),
            "boltz_end_flux": (i, [vp, vp, i64, vp, vp, i, i, d, vp, vp]),
            "boltz_set_async": (i, [vp, i]),
            "boltz_set_schedule": (i, [vp, i]),
            "boltz_schedule_terms": (i, [vp, C.POINTER(i64), C.POINTER(i64)]),
            "boltz_conv_kernel": (C.c_char_p, [vp]),
            "boltz_create_transform": (i, [i, d, i, C.POINTER(vp)]),
            "boltz_sync": (i, [vp, vp]),
            "boltz_set_timing": (i, [vp, i]),
            "boltz_get_timing": (i, [vp, vp, vp, i, i]),
            "boltz_fp64_peak": (i, [i, d, dp]),
            "boltz_generate_table": (i, [i, d, d, d, d, i, vp, i]),
            "boltz_weight": (d, [d, d, d, vp, vp, i]),
            "boltz_save_table": (i, [C.c_char_p, i, d, d, d, d, i, vp]),
            "boltz_load_table": (i, [C.c_char_p, i, d, d, d, d, i, vp]),
            "boltz_halo_unique_id": (i, [vp]),
            "boltz_halo_create": (i, [i, i, vp, i, C.POINTER(vp)]),
            "boltz_halo_destroy": (i, [vp]),
            "boltz_halo_exchange": (i, [vp, vp, i64, i64, vp]),
            "boltz_halo_allreduce_sum": (i, [vp, vp, i64, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc:
        msg = lib().boltz_last_error().decode()
        raise _ERR.get(rc, BoltzError)(msg, rc)


# ----------------------------------------------------------------- grid
@dataclass
class VelocityGrid:
    """Cubic velocity lattice + Fourier dual (velocity_grid.hpp:8-47)."""
    n: int
    half_width: float
    dv: float
    dzeta: float
    v_nodes: np.ndarray
    zeta_nodes: np.ndarray
    axis_coeff: np.ndarray

    @staticmethod
    def create(n: int, half_width: float) -> "VelocityGrid":
        # velocity_grid.cpp:11-32
        if n < 4 or n % 2 != 0:
            raise ConfigError(f"velocity grid: N must be even and >= 4, got {n}")
        if not half_width > 0.0:
            raise ConfigError(f"velocity grid: L must be positive, got {half_width}")
        dv = 2.0 * half_width / n
        dz = math.pi / half_width
        k = np.arange(n)
        coeff = np.ones(n)
        coeff[0] = coeff[-1] = 0.5
        return VelocityGrid(n, float(half_width), dv, dz, dv * (k - n // 2), dz * (k - n // 2), coeff)

    def size(self) -> int:
        return self.n ** 3

    def flat(self, i, j, k) -> int:
        return (i * self.n + j) * self.n + k

    def coeff3(self, i, j, k) -> float:
        return self.axis_coeff[i] * self.axis_coeff[j] * self.axis_coeff[k]

    def vel_weight(self, i, j, k) -> float:
        return self.coeff3(i, j, k) * self.dv ** 3

    def fourier_weight(self, i, j, k) -> float:
        return self.coeff3(i, j, k) * self.dzeta ** 3

    def velocities(self) -> np.ndarray:
        """(N^3, 3) node velocities in flat order."""
        v = self.v_nodes
        V1, V2, V3 = np.meshgrid(v, v, v, indexing="ij")
        return np.stack([V1.ravel(), V2.ravel(), V3.ravel()], axis=1)

    def vel_weights(self) -> np.ndarray:
        c = self.axis_coeff
        return (c[:, None, None] * c[None, :, None] * c[None, None, :]).ravel() * self.dv ** 3


@dataclass
class KernelSpec:
    """Collision kernel |u|^lambda, isotropic b = 1/(4 pi)."""
    lam: float = 1.0
    beta: float = 1.0
    r0: Optional[float] = None
    panels: int = 64  # Gauss-Legendre panels for 0 < lambda < 1

    def radius(self, grid: VelocityGrid) -> float:
        return grid.half_width if self.r0 is None else self.r0  # r0 = L


# ------------------------------------------------------------- weights
def weight(kernel: KernelSpec, xi, zeta, r0: float) -> float:
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    zeta = np.ascontiguousarray(zeta, dtype=np.float64)
    return lib().boltz_weight(kernel.lam, kernel.beta, r0, xi.ctypes.data, zeta.ctypes.data, kernel.panels)


def generate_table(grid: VelocityGrid, kernel: KernelSpec, nthreads: int = 0) -> np.ndarray:
    """Dense zeta-major table G[k][m], N^6 doubles."""
    n = grid.n
    G = np.empty(n ** 6, dtype=np.float64)
    _check(lib().boltz_generate_table(n, grid.half_width, kernel.lam, kernel.beta, kernel.radius(grid),
                                      kernel.panels, G.ctypes.data, nthreads))
    return G


def save_table(path, grid: VelocityGrid, kernel: KernelSpec, G: np.ndarray) -> None:
    G = np.ascontiguousarray(G, dtype=np.float64)
    _check(lib().boltz_save_table(str(path).encode(), grid.n, grid.half_width, kernel.lam, kernel.beta,
                                  kernel.radius(grid), kernel.panels, G.ctypes.data))


def load_table(path, grid: VelocityGrid, kernel: KernelSpec) -> np.ndarray:
    G = np.empty(grid.n ** 6, dtype=np.float64)
    _check(lib().boltz_load_table(str(path).encode(), grid.n, grid.half_width, kernel.lam, kernel.beta,
                                  kernel.radius(grid), kernel.panels, G.ctypes.data))
    return G


def fp64_peak(device: int = 0, seconds: float = 0.5) -> float:
    """Measured DFMA throughput of the device (TFLOP/s)."""
    t = C.c_double()
    _check(lib().boltz_fp64_peak(device, seconds, C.byref(t)))
    return t.value


# --------------------------------------------------------------- halo
class NcclHalo:
    """The C ABI's NCCL halo (boltz_halo_*, csrc/halo.cpp): one grouped
    send/recv of the two edge cells per neighbour on the caller's stream, plus
    the ledger all-reduce.  Rank 0's communicator id is broadcast over
    torch.distributed (any backend).  Unlike torch.distributed P2P it can be
    captured in a CUDA graph, so Solver1D.run replays multi-rank steps too.
    Import torch before creating one (the library then binds torch's NCCL)."""

    def __init__(self, rank: int, world: int, device: int = 0):
        import torch  # noqa: F401  (NCCL binding order, csrc/halo.cpp)
        self.rank, self.world = rank, world
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _check(lib().boltz_halo_unique_id(uid))
        if world > 1:
            import torch.distributed as dist
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0)
            uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib().boltz_halo_create(rank, world, uid, device, C.byref(h)))
        self._h = h

    def exchange(self, field) -> int:
        """Refresh the 2+2 halo ghosts of a (ncl+4, N^3) CUDA field (collective)."""
        import torch
        s = torch.cuda.current_stream(field.device).cuda_stream
        _check(lib().boltz_halo_exchange(self._h, C.c_void_p(field.data_ptr()), field.shape[0] - 4, field.shape[1],
                                         C.c_void_p(s)))
        return (self.rank > 0) + (self.rank < self.world - 1)

    def all_reduce(self, t) -> None:
        """In-place sum over ranks of a float64 CUDA tensor (collective)."""
        import torch
        s = torch.cuda.current_stream(t.device).cuda_stream
        _check(lib().boltz_halo_allreduce_sum(self._h, C.c_void_p(t.data_ptr()), t.numel(), C.c_void_p(s)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _check(lib().boltz_halo_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ operator
def _is_torch(x):
    return type(x).__module__.startswith("torch")


class CollisionOperator:
    """Batched GPU collision operator on one device.

    Replaces, for a batch of spatial cells, the reference's
    SpectralTransform (forward/inverse, fourier.hpp:36-41), evaluate_qhat,
    conserve and collide and collision_rk2
    (SPEC.md:383-391).  A batch is (ncells, N^3) real / complex, flat index
    (i1*N+i2)*N+i3.  The table is copied to HBM (folded, pair-symmetric
    layout) at construction; the host copy may be dropped afterwards.
    Not thread-safe (like SpectralTransform, fourier.hpp:24-25).
    """

    def __init__(self, grid: VelocityGrid, kernel: KernelSpec, table: Optional[np.ndarray], device: int = 0):
        """table: the dense zeta-major N^6 host table (generate_table/load_table),
        or None to evaluate it on the device (boltz_create_generated)."""
        self.grid, self.kernel, self.device = grid, kernel, device
        h = C.c_void_p()
        if table is None:
            _check(lib().boltz_create_generated(grid.n, grid.half_width, kernel.lam, kernel.beta,
                                                kernel.radius(grid), kernel.panels, device, C.byref(h)))
        else:
            table = np.ascontiguousarray(table, dtype=np.float64)
            if table.size != grid.n ** 6:
                raise ConfigError(f"weight table has {table.size} entries, expected N^6 = {grid.n ** 6}")
            _check(lib().boltz_create(grid.n, grid.half_width, kernel.lam, kernel.beta, kernel.radius(grid),
                                      table.ctypes.data, device, C.byref(h)))
        self._h = h

    @classmethod
    def generated(cls, grid: VelocityGrid, kernel: KernelSpec, device: int = 0) -> "CollisionOperator":
        """Context whose weight table is generated on the GPU (no host N^6 table)."""
        return cls(grid, kernel, None, device)

    def close(self):
        if getattr(self, "_h", None):
            lib().boltz_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def memory_bytes(self):
        a, b = C.c_int64(), C.c_int64()
        _check(lib().boltz_memory_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def moments(self, f):
        """compute_moments per cell: (ncells, 7) =
        rho, rho*V (3), rho*e, T, H."""
        f = self._prep(f)
        nc = self._ncells(f, self.grid.size())
        out = self._alloc_like(f, (nc, 7))
        (pf, po), mem, s = self._args(f, out)
        _check(lib().boltz_moments_batch(self._h, pf, po, nc, mem, s))
        return out

    def marginal(self, f):
        """marginal_distribution per cell: (ncells, N) = g(v1) = sum_{v2,v3} f w2 w3."""
        f = self._prep(f)
        nc = self._ncells(f, self.grid.size())
        out = self._alloc_like(f, (nc, self.grid.n))
        (pf, po), mem, s = self._args(f, out)
        _check(lib().boltz_marginal_batch(self._h, pf, po, nc, mem, s))
        return out

    def schedule_terms(self):
        """(plain, mirror) executed K2 terms per cell eval (mirror 0 when the
        Hermitian mirror schedule is not active)."""
        a, b = C.c_int64(), C.c_int64()
        _check(lib().boltz_schedule_terms(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def conv_kernel(self) -> str:
        """The K2 kernel(s) collide / RK2 run under the current schedule."""
        return lib().boltz_conv_kernel(self._h).decode()

    def set_schedule(self, schedule="throughput"):
        """K2 schedule: "throughput" (default), "latency" (each row's entries in 4
        fixed segments on 4 warps: small batches, N <= 16), "latency8" (8
        segments: a few cells), "cell" (lane = output k3: one or a few cells,
        N <= 16), "auto" (picked per call from the batch size: cell up to 4
        cells, latency8 up to 64, latency up to 256, else throughput), or the
        ABI's integer 0..6.  Bitwise reproducible within a schedule; schedules
        differ by round-off."""
        code = {"throughput": 0, "latency": 1, "latency8": 2, "cell": 5, "auto": 6}.get(schedule, schedule)
        _check(lib().boltz_set_schedule(self._h, int(code)))

    # -- asynchronous mode (CUDA-graph capturable device calls)
    def set_async(self, enable: bool = True):
        """Device-pointer calls stop synchronising; errors surface at sync()."""
        _check(lib().boltz_set_async(self._h, int(enable)))

    def sync(self, stream=None):
        """Synchronise and raise NumericError for any non-finite value seen since the last sync."""
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(self.device).cuda_stream
            except Exception:
                stream = None
        _check(lib().boltz_sync(self._h, stream))

    # -- measurement hooks (bench.py)
    KINDS = ("conv", "fft", "project", "layout", "transport")

    def set_timing(self, enable: bool = True):
        _check(lib().boltz_set_timing(self._h, int(enable)))

    def timing(self, reset: bool = False):
        """({kind: ms}, {kind: launches}) accumulated since the last reset."""
        ms = np.zeros(5)
        cnt = np.zeros(5, dtype=np.int64)
        _check(lib().boltz_get_timing(self._h, ms.ctypes.data, cnt.ctypes.data, 5, int(reset)))
        return dict(zip(self.KINDS, ms.tolist())), dict(zip(self.KINDS, cnt.tolist()))

    # -- argument plumbing
    def _ncells(self, x, per_cell):
        n = x.numel() if _is_torch(x) else x.size
        if n % per_cell:
            raise ConfigError(f"array of {n} values is not a whole number of cells ({per_cell} per cell)")
        return n // per_cell

    def _args(self, *arrays, complex_idx=()):
        """Pointers, memory kind and stream for a call. Device arrays must be
        contiguous CUDA tensors on this operator's device, complex128 at the
        positions in `complex_idx` and float64 elsewhere."""
        if all(_is_torch(a) for a in arrays):
            import torch
            for i, a in enumerate(arrays):
                want = torch.complex128 if i in complex_idx else torch.float64
                if not (a.is_cuda and a.is_contiguous()):
                    raise ConfigError("device arrays must be contiguous CUDA tensors")
                if a.dtype != want:
                    raise ConfigError(f"argument {i}: expected a {want} tensor, got {a.dtype}")
                if a.device.index != self.device:
                    raise ConfigError(f"argument {i} lives on cuda:{a.device.index}, the operator on cuda:{self.device}")
            return [a.data_ptr() for a in arrays], MEM_DEVICE, torch.cuda.current_stream(arrays[0].device).cuda_stream
        if any(_is_torch(a) for a in arrays):
            raise ConfigError("mix of host and device arrays")
        for i, a in enumerate(arrays):
            want = np.complex128 if i in complex_idx else np.float64
            if a.dtype != want:
                raise ConfigError(f"argument {i}: expected a {np.dtype(want)} array, got {a.dtype}")
        return [a.ctypes.data for a in arrays], MEM_HOST, None

    def _alloc_like(self, x, shape, complex_=False):
        if _is_torch(x):
            import torch
            return torch.empty(shape, dtype=torch.complex128 if complex_ else torch.float64, device=x.device)
        return np.empty(shape, dtype=np.complex128 if complex_ else np.float64)

    @staticmethod
    def _host(x, dtype):
        return np.ascontiguousarray(x, dtype=dtype)

    def _prep(self, x, complex_=False):
        if _is_torch(x):
            return x.contiguous()  # dtype and device are checked by _args
        if not complex_ and np.iscomplexobj(x):
            raise ConfigError("expected real data, got a complex array")
        return self._host(x, np.complex128 if complex_ else np.float64)

    # -- reference operations, batched
    def forward(self, f):
        """SpectralTransform::forward (fourier.hpp:36): real -> complex."""
        f = self._prep(f)
        n3 = self.grid.size()
        nc = self._ncells(f, n3)
        out = self._alloc_like(f, (nc, n3), complex_=True)
        (pf, po), mem, s = self._args(f, out, complex_idx=(1,))
        _check(lib().boltz_forward_batch(self._h, pf, po, nc, mem, s))
        return out

    def inverse(self, g):
        """SpectralTransform::inverse (fourier.hpp:38-41) -> (real, max_imag per cell)."""
        g = self._prep(g, complex_=True)
        n3 = self.grid.size()
        nc = self._ncells(g, n3)
        out = self._alloc_like(g, (nc, n3))
        mi = self._alloc_like(g, (nc,))
        (pg, po, pm), mem, s = self._args(g, out, mi, complex_idx=(0,))
        _check(lib().boltz_inverse_batch(self._h, pg, po, pm, nc, mem, s))
        return out, mi

    def evaluate_qhat(self, fhat):
        """evaluate_qhat, complex -> complex."""
        fhat = self._prep(fhat, complex_=True)
        n3 = self.grid.size()
        nc = self._ncells(fhat, n3)
        out = self._alloc_like(fhat, (nc, n3), complex_=True)
        (pf, po), mem, s = self._args(fhat, out, complex_idx=(0, 1))
        _check(lib().boltz_qhat_batch(self._h, pf, po, nc, mem, s))
        return out

    def conserve(self, q_raw):
        """conserve."""
        q_raw = self._prep(q_raw)
        n3 = self.grid.size()
        nc = self._ncells(q_raw, n3)
        out = self._alloc_like(q_raw, (nc, n3))
        (pq, po), mem, s = self._args(q_raw, out)
        _check(lib().boltz_conserve_batch(self._h, pq, po, nc, mem, s))
        return out

    def collide(self, f, epsilon: float = 1.0, with_max_imag: bool = False):
        """collide: (1/eps) P_N(inverse(qhat(forward(f))))."""
        if not epsilon > 0.0:
            raise ConfigError("collide: epsilon must be positive")
        f = self._prep(f)
        n3 = self.grid.size()
        nc = self._ncells(f, n3)
        out = self._alloc_like(f, (nc, n3))
        if with_max_imag:
            mi = self._alloc_like(f, (nc,))
            (pf, po, pm), mem, s = self._args(f, out, mi)
        else:
            mi = None
            (pf, po), mem, s = self._args(f, out)
            pm = None
        _check(lib().boltz_collide_batch(self._h, pf, po, nc, 1.0 / epsilon, pm, mem, s))
        return (out, mi) if with_max_imag else out

    def collision_rk2(self, f, dt: float, epsilon: float = 1.0):
        """collision_rk2, IN PLACE on f (numpy or torch)."""
        if not dt > 0.0 or not epsilon > 0.0:
            raise ConfigError("collision_rk2: dt and epsilon must be positive")
        if not _is_torch(f) and not (isinstance(f, np.ndarray) and f.dtype == np.float64 and f.flags.c_contiguous):
            raise ConfigError("collision_rk2 works in place: pass a C-contiguous float64 array")
        n3 = self.grid.size()
        nc = self._ncells(f, n3)
        (pf,), mem, s = self._args(f)
        _check(lib().boltz_rk2_batch(self._h, pf, nc, dt, 1.0 / epsilon, mem, s))
        return f

    # -- transport (device tensors only)
    def transport_step(self, field, out, x_ext, dx_ext, dt, wall_left=False, wall_right=False, base=None,
                       alpha=0.0, rows=None):
        """transport_step on a (ncl+4, N^3) device field:
        out = alpha*base + (1-alpha)*step(field) (base=None: the plain step).
        rows=(c_begin, c_end): only those interior rows (boltz_transport_step_range)."""
        ncl = field.shape[0] - 4
        arrs = (field, out, x_ext, dx_ext) + ((base,) if base is not None else ())
        ptrs, mem, s = self._args(*arrs)
        if mem != MEM_DEVICE:
            raise ConfigError("transport_step takes CUDA tensors")
        pb = ptrs[4] if base is not None else None
        if rows is None:
            _check(lib().boltz_transport_step(self._h, ptrs[0], pb, alpha, ptrs[1], ncl, ptrs[2], ptrs[3], dt,
                                              int(wall_left), int(wall_right), s))
        else:
            _check(lib().boltz_transport_step_range(self._h, ptrs[0], pb, alpha, ptrs[1], ncl, ptrs[2], ptrs[3], dt,
                                                    int(wall_left), int(wall_right), int(rows[0]), int(rows[1]), s))
        return out

    def end_flux(self, field, x_ext, dx_ext, acc, coef, wall_left=False, wall_right=False):
        """Boundary-flux ledger: acc (5-double CUDA tensor) += coef * (F(right end
        face) - F(left end face)) of (mass, momentum 1-3, energy)."""
        ncl = field.shape[0] - 4
        ptrs, mem, s = self._args(field, x_ext, dx_ext, acc)
        if mem != MEM_DEVICE:
            raise ConfigError("end_flux takes CUDA tensors")
        _check(lib().boltz_end_flux(self._h, ptrs[0], ncl, ptrs[1], ptrs[2], int(wall_left), int(wall_right), coef,
                                    ptrs[3], s))
        return acc

    def fill_boundary(self, field, x_ext, side, kind, Tw=1.0, Vw=(0.0, 0.0, 0.0)):
        """Ghost fill at a physical end: kind 0 extrapolation, 1 diffuse wall. Returns sigma_w."""
        ncl = field.shape[0] - 4
        (pf, px), mem, s = self._args(field, x_ext)
        if mem != MEM_DEVICE:
            raise ConfigError("fill_boundary takes CUDA tensors")
        vw = np.ascontiguousarray(Vw, dtype=np.float64)
        sig = C.c_double()
        _check(lib().boltz_fill_boundary(self._h, pf, ncl, px, side, kind, Tw, vw.ctypes.data, C.byref(sig), s))
        return sig.value

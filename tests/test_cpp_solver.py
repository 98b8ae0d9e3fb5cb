"""The C++ host driver (include/boltz_solver.hpp: Solver1D, plan_decomposition,
loopback and NCCL halo, over the C ABI) compiles on CPU and, on a GPU,
reproduces the Python driver (paper_1301_4195_b200/solver.py) bit for bit --
the same kernels in the same order -- for 1 rank with an NCCL communicator and
for 3 loopback ranks (decomposition transparency), and with
CUDA-graph replay of the Strang step (7 steps = 1 eager + 2 replays), and with
the halo fused into the transport kernels (PeerGroup, 3 and 5 ranks with their
own contexts and streams on one device)."""
import pathlib
import subprocess

import numpy as np
import pytest

from paper_1301_4195_b200.build import LIB, build

REPO = pathlib.Path(__file__).resolve().parent.parent
EXE = REPO / "tests" / "cpp" / "solver_demo"


def _compile():
    build()
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(REPO / "include"), "-I", "/usr/local/cuda/include",
                    "-o", str(EXE), str(REPO / "tests" / "cpp" / "solver_demo.cpp"), str(LIB),
                    "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIB.parent}:/usr/local/cuda/lib64"],
                   check=True)


def test_cpp_solver_compiles():
    _compile()
    assert EXE.exists()


def test_halo_abi_without_gpu():
    """The NCCL binding is lazy (dlopen): a unique id needs no GPU; bad
    arguments are ConfigErrors.  torch is imported first, as in any process
    that uses both: the library then binds torch's libnccl.so.2 (RTLD_NOLOAD)
    instead of loading the system one under the same soname."""
    import ctypes
    import torch  # noqa: F401
    build()
    L = ctypes.CDLL(str(LIB))
    buf = (ctypes.c_ubyte * 128)()
    assert L.boltz_halo_unique_id(buf) == 0 and any(bytes(buf))
    out = ctypes.c_void_p()
    assert L.boltz_halo_create(2, 2, buf, 0, ctypes.byref(out)) == 2  # rank >= world
    assert L.boltz_halo_exchange(None, None, 4, 8, None) == 2
    assert L.boltz_halo_exchange_loopback(None, None, 0, 8, None) == 2


@pytest.mark.gpu
def test_cpp_solver_matches_python_driver(gpu, tmp_path):
    import torch
    from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
    from paper_1301_4195_b200.solver import Boundary, Solver1D
    _compile()
    n, L, lam, Tw, nx, steps = 8, 5.0, 1.0, 2.0, 10, 7
    grid = VelocityGrid.create(n, L)
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    f0 = scenarios.mixture_cells(grid, nx, seed=17)
    x.tofile(tmp_path / "x.bin")
    dx.tofile(tmp_path / "dx.bin")
    np.ascontiguousarray(f0).tofile(tmp_path / "f0.bin")
    with CollisionOperator.generated(grid, KernelSpec(lam)) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw), right=Boundary("extrap"))
        dt = s.cfl_dt()
        for _ in range(steps):
            s.strang_step(dt)
        ref = s.interior.cpu().numpy()
    torch.cuda.synchronize()
    for mode, nranks in [("nccl", 1), ("nccl_overlap", 1), ("loopback", 3), ("graph", 1), ("peer", 3), ("peer", 5)]:
        r = subprocess.run([str(EXE), str(tmp_path), str(n), repr(L), repr(lam), repr(Tw), repr(dt), str(steps),
                            str(nranks), mode], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        got = np.fromfile(tmp_path / f"out_{mode}_{nranks}.bin").reshape(nx, -1)
        assert np.array_equal(got, ref), (mode, np.abs(got - ref).max())
        assert "ledger mass" in r.stdout


@pytest.mark.gpu
def test_cpp_solver_single_stage_matches_python_driver(gpu, tmp_path):
    """TransportScheme::SingleStage in the C++ driver equals
    the Python driver's transport_scheme="single_stage" bit for bit, for the
    loopback, graph-replay and fused peer-halo modes."""
    import torch
    from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, scenarios
    from paper_1301_4195_b200.solver import Boundary, Solver1D
    _compile()
    n, L, lam, Tw, nx, steps = 8, 5.0, 1.0, 2.0, 10, 7
    grid = VelocityGrid.create(n, L)
    x, dx = scenarios.geometric_grid(nx, 2.0, 1.1)
    f0 = scenarios.mixture_cells(grid, nx, seed=19)
    x.tofile(tmp_path / "x.bin")
    dx.tofile(tmp_path / "dx.bin")
    np.ascontiguousarray(f0).tofile(tmp_path / "f0.bin")
    with CollisionOperator.generated(grid, KernelSpec(lam)) as op:
        s = Solver1D(op, x, dx, f0, left=Boundary("wall", Tw), right=Boundary("extrap"),
                     transport_scheme="single_stage")
        dt = 0.5 * s.cfl_dt()
        for _ in range(steps):
            s.strang_step(dt)
        ref = s.interior.cpu().numpy()
    torch.cuda.synchronize()
    for mode, nranks in [("loopback", 3), ("graph", 1), ("peer", 3)]:
        r = subprocess.run([str(EXE), str(tmp_path), str(n), repr(L), repr(lam), repr(Tw), repr(dt), str(steps),
                            str(nranks), mode, "single"], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        got = np.fromfile(tmp_path / f"out_{mode}_{nranks}_single.bin").reshape(nx, -1)
        assert np.array_equal(got, ref), (mode, np.abs(got - ref).max())

"""The drop-in in the reference's own types:
paper_1301_4195_b200/shim/fourier_cuda.cpp implements boltz::SpectralTransform
exactly as the UNMODIFIED proj/include/boltz/fourier.hpp:28-52 declares it,
shim/collision_cuda.cpp the SPEC collision operations (SPEC.md:186-212,
383-391) with the reference's exceptions (errors.hpp:9-35), and
include/boltz_cuda.hpp maps its errors onto boltz::Error when built inside the
reference tree.  tests/cpp/ref_shim_demo links them with the reference's own
velocity_grid.cpp (compiled in place, never copied).  The binary is built here
(build_shim, from /root/reference); the GPU box runs the prebuilt binary."""
import pathlib
import subprocess

import numpy as np
import pytest

from conftest import rel_max, table

REPO = pathlib.Path(__file__).resolve().parent.parent
EXE = REPO / "tests" / "cpp" / "ref_shim_demo"
REF = pathlib.Path("/root/reference/proj/include/boltz/fourier.hpp")


def test_shim_builds_against_unmodified_reference_header():
    if not REF.exists():
        if not EXE.exists():
            pytest.skip("no reference tree and no prebuilt ref_shim_demo")
        return
    from paper_1301_4195_b200.build import build_shim
    assert build_shim(force=True) == EXE and EXE.exists()


@pytest.mark.gpu
@pytest.mark.parametrize("n,L,lam", [(8, 5.0, 1.0), (16, 6.0, 0.0)])
def test_reference_types_drop_in_vs_oracle(gpu, O, tmp_path, n, L, lam):
    from paper_1301_4195_b200 import VelocityGrid, scenarios
    from paper_1301_4195_b200.build import build_shim
    exe = build_shim()
    assert exe is not None and exe.exists(), "tests/cpp/ref_shim_demo was not built (needs /root/reference once)"
    grid = VelocityGrid.create(n, L)
    f = scenarios.mixture_cells(grid, 5, seed=101)
    G = table(n, L, lam)
    f.tofile(tmp_path / "f.bin")
    np.ascontiguousarray(G).tofile(tmp_path / "G.bin")
    r = subprocess.run([str(exe), str(tmp_path), str(n), repr(L), repr(lam)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    n3 = n ** 3
    fhat = np.fromfile(tmp_path / "fhat.bin", dtype=np.complex128)
    ref_fh = O.forward(n, L, f[0])
    assert rel_max(fhat, ref_fh) < 1e-12
    back = np.fromfile(tmp_path / "back.bin")
    rb, rmi = O.inverse(n, L, ref_fh)
    assert rel_max(back, rb) < 1e-12
    assert abs(np.fromfile(tmp_path / "max_imag.bin")[0] - rmi) <= 1e-12 * np.abs(rb).max() + 1e-300
    qhat = np.fromfile(tmp_path / "qhat.bin", dtype=np.complex128)
    assert rel_max(qhat, O.evaluate_qhat(n, L, G, ref_fh)) < 1e-10
    q = np.fromfile(tmp_path / "q.bin").reshape(5, n3)
    rk = np.fromfile(tmp_path / "rk2.bin").reshape(5, n3)
    ref_rk = O.collision_rk2(n, L, G, f, 0.01)
    for c in range(5):
        rq, _ = O.collide(n, L, G, f[c])
        assert rel_max(q[c], rq) < 1e-10
        assert rel_max(rk[c] - f[c], ref_rk[c] - f[c]) < 1e-9
    for line in ("collide(NaN): NumericError category 4", "collision_rk2(NaN): NumericError category 4",
                 "collide(ragged): ConfigError category 2", "forward(short span): ConfigError category 2",
                 "SpectralTransform(N=10): ConfigError category 2", "VelocityGrid(N=5): ConfigError category 2",
                 "cuda::CollisionOperator::collide(NaN): NumericError category 4", "ref_shim_demo ok"):
        assert line in out, out

"""Host-side logic and the C-ABI boundary (CPU only, no compute calls on a GPU).

* the library loads and exports every entry point include/boltz_cuda.h declares;
* the product's host weight generator equals the oracle's table;
* save/load_table round trip and its error categories;
* VelocityGrid mirror vs the reference-pinned golden grid;
* no silent CPU fallback: without a GPU the operator raises.
"""
import json
import pathlib
import re

import numpy as np
import pytest

from paper_1301_4195_b200 import (ConfigError, CudaError, IoError, KernelSpec, VelocityGrid, generate_table, lib,
                                  load_table, save_table, weight)
from paper_1301_4195_b200.build import LIB, build

REPO = pathlib.Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def test_library_exports_every_declared_symbol():
    hdr = (REPO / "include" / "boltz_cuda.h").read_text()
    names = set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(boltz_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 20, names
    L = lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    # exported with C linkage (no mangling) and built for sm_100a
    info = L.boltz_build_info().decode()
    assert "sm_100a" in info


def test_cubin_targets_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(LIB)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,L,lam", [(6, 4.0, 1.0), (8, 5.0, 0.0), (8, 5.0, 1.0)])
def test_host_table_equals_oracle(O, n, L, lam):
    G = generate_table(VelocityGrid.create(n, L), KernelSpec(lam))
    Go = O.generate_table(n, L, lam)
    assert np.abs(G - Go).max() <= 1e-13 * np.abs(Go).max()


def test_host_table_general_lambda_matches_oracle_quadrature(O):
    n, L = 4, 3.0
    G = generate_table(VelocityGrid.create(n, L), KernelSpec(0.5, panels=32))
    Go = O.generate_table(n, L, 0.5, panels=32)
    assert np.abs(G - Go).max() <= 1e-12 * np.abs(Go).max()


def test_host_table_thread_invariant():
    g = VelocityGrid.create(8, 5.0)
    from paper_1301_4195_b200.boltz import generate_table as gt
    assert np.array_equal(gt(g, KernelSpec(1.0), nthreads=1), gt(g, KernelSpec(1.0), nthreads=7))


def test_weight_point_values(O):
    dz = np.pi / 5.0
    for xi, ze in [((dz, 0, 0), (0, dz, 0)), ((0, 0, 0), (0, 0, 0)), ((dz, dz, 0), (2 * dz, 2 * dz, 0))]:
        for lam in (0.0, 1.0):
            a = weight(KernelSpec(lam), xi, ze, 5.0)
            b = O.weight_closed_form(lam, 1.0, 5.0, np.array(xi, float), np.array(ze, float))
            assert abs(a - b) <= 1e-13 * max(1.0, abs(b))


def test_table_cache_round_trip_and_errors(tmp_path):
    g = VelocityGrid.create(4, 3.0)
    k = KernelSpec(1.0)
    G = generate_table(g, k)
    p = tmp_path / "w.tbl"
    save_table(p, g, k, G)
    assert np.array_equal(load_table(p, g, k), G)
    with pytest.raises(ConfigError, match="N expected 6"):  # SPEC.md:142 names both values
        load_table(p, VelocityGrid.create(6, 3.0), k)
    with pytest.raises(ConfigError, match="lambda"):
        load_table(p, g, KernelSpec(0.0))
    raw = p.read_bytes()
    (tmp_path / "t.tbl").write_bytes(raw[:-8])
    with pytest.raises(IoError, match="truncated"):
        load_table(tmp_path / "t.tbl", g, k)
    (tmp_path / "c.tbl").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(IoError, match="corrupt header"):
        load_table(tmp_path / "c.tbl", g, k)
    with pytest.raises(IoError):
        load_table(tmp_path / "missing.tbl", g, k)


def test_velocity_grid_mirror_matches_reference_golden():
    data = json.loads((REPO / "tests" / "golden" / "grid_ref.json").read_text())
    for gd in data["grids"]:
        g = VelocityGrid.create(gd["n"], gd["L"])
        assert g.dv == gd["dv"] and g.dzeta == gd["dzeta"]
        assert np.array_equal(g.v_nodes, gd["v"]) and np.array_equal(g.zeta_nodes, gd["zeta"])
        assert np.array_equal(g.axis_coeff, gd["coeff"])
        assert g.flat(1, 2, 3) == gd["flat_123"]
    for e in data["errors"]:
        with pytest.raises(ConfigError):
            VelocityGrid.create(e["n"], e["L"])


def test_generate_table_rejects_bad_input():
    with pytest.raises(ConfigError):
        generate_table(VelocityGrid(5, 1.0, 0.4, 3.0, np.zeros(5), np.zeros(5), np.ones(5)), KernelSpec(1.0))
    with pytest.raises(ConfigError):
        generate_table(VelocityGrid.create(4, 1.0), KernelSpec(1.5))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1301_4195_b200 import CollisionOperator
    g = VelocityGrid.create(4, 3.0)
    with pytest.raises(CudaError):
        CollisionOperator(g, KernelSpec(1.0), generate_table(g, KernelSpec(1.0)))


def test_unsupported_n_is_config_error():
    from paper_1301_4195_b200 import CollisionOperator
    g = VelocityGrid.create(10, 3.0)
    with pytest.raises(ConfigError, match="no compiled kernel"):
        CollisionOperator(g, KernelSpec(1.0), np.zeros(10 ** 6))


def test_scenarios_portable_rng():
    from paper_1301_4195_b200 import scenarios
    # vectorised SplitMix64 == a scalar pure-Python SplitMix64 (Python ints, explicit 64-bit masks)
    M = (1 << 64) - 1

    def scalar(seed, count):
        out, x = [], seed
        for _ in range(count):
            x = (x + 0x9E3779B97F4A7C15) & M
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
            out.append(z ^ (z >> 31))
        return out

    for seed in (0, 1, 4195, 2 ** 63 + 12345):
        assert [int(v) for v in scenarios.splitmix64(seed, 50)] == scalar(seed, 50)
    assert hex(int(scenarios.splitmix64(0, 1)[0])) == "0xe220a8397b1dcdaf"
    u = scenarios.uniform(1, 1000)
    assert u.min() >= 0 and u.max() < 1
    g = VelocityGrid.create(8, 5.0)
    a = scenarios.mixture_cells(g, 5, seed=3)
    b = scenarios.mixture_cells(g, 2, seed=3, first=3)
    assert np.array_equal(a[3:], b)  # cell i depends only on (seed, i)


def test_geometric_grid_cfg3():
    from paper_1301_4195_b200 import scenarios
    x, dx = scenarios.geometric_grid(256, 20.0, 1.02)
    assert abs(dx.sum() - 20.0) < 1e-12 and abs(dx[0] - 2.530e-3) < 1e-5
    assert np.allclose(np.diff(x), 0.5 * (dx[1:] + dx[:-1]), rtol=0, atol=1e-13)
    xe, dxe = scenarios.extend_ghosts(x, dx)
    assert len(xe) == 260 and np.allclose(np.diff(xe), 0.5 * (dxe[1:] + dxe[:-1]), atol=1e-13)

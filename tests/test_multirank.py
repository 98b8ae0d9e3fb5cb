"""Multi-rank halo exchange and decomposition on CPU (gloo, world_size 2 and 4).

The GPU run uses the same TorchHalo over NCCL; here the ranks are CPU
processes (SPEC.md:452-453 examples, SPEC.md:465 transparency contract)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1301_4195_b200.solver import LoopbackHalo, TorchHalo, plan_decomposition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nx, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = plan_decomposition(nx, world)
        start, ncl = plan[rank]
        rng = np.random.default_rng(123)
        glob = rng.random((nx, m))
        glob[:, 0] = np.arange(nx)  # index-valued column
        field = torch.full((ncl + 4, m), -1.0, dtype=torch.float64)
        field[2:ncl + 2] = torch.from_numpy(glob[start:start + ncl])
        pairs = TorchHalo(rank, world).exchange(field)
        q.put((rank, start, ncl, pairs, field.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nx", [(2, 10), (4, 13)])
def test_torch_halo_gloo(world, nx):
    m = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(123)
    glob = rng.random((nx, m))
    glob[:, 0] = np.arange(nx)
    for rank, start, ncl, pairs, field in res:
        assert pairs == (1 if rank in (0, world - 1) else 2)
        if rank > 0:  # left ghosts = the left neighbour's two rightmost interior cells
            assert np.array_equal(field[0:2], glob[start - 2:start])
        else:
            assert np.all(field[0:2] == -1.0)  # physical end: filled by boundary rules, not messages
        if rank < world - 1:
            assert np.array_equal(field[ncl + 2:ncl + 4], glob[start + ncl:start + ncl + 2])
            assert list(field[ncl + 2:ncl + 4, 0]) == [start + ncl, start + ncl + 1]
        else:
            assert np.all(field[ncl + 2:] == -1.0)


def test_loopback_matches_global_ghosts():
    """n=4 loopback exchange == ghosts of the single global array."""
    nx, m, world = 13, 5, 4
    rng = np.random.default_rng(7)
    glob = rng.random((nx, m))
    plan = plan_decomposition(nx, world)
    fields = []
    for s, c in plan:
        f = np.zeros((c + 4, m))
        f[2:c + 2] = glob[s:s + c]
        fields.append(f)
    LoopbackHalo.exchange_all(fields)
    for (s, c), f in zip(plan, fields):
        if s > 0:
            assert np.array_equal(f[0:2], glob[s - 2:s])
        if s + c < nx:
            assert np.array_equal(f[c + 2:c + 4], glob[s + c:s + c + 2])


def test_plan_decomposition_contract():
    assert plan_decomposition(10, 2) == [(0, 5), (5, 5)]
    assert [c for _, c in plan_decomposition(10, 3)] == [4, 3, 3]
    for nx in range(1, 40):
        for n in range(1, min(nx, 9) + 1):
            p = plan_decomposition(nx, n)
            assert sum(c for _, c in p) == nx and max(c for _, c in p) - min(c for _, c in p) <= 1
            assert all(p[i][0] + p[i][1] == p[i + 1][0] for i in range(n - 1))
    from paper_1301_4195_b200 import ConfigError
    with pytest.raises(ConfigError):
        plan_decomposition(2, 3)


def test_predict_speedup_limits():
    """SPEC acceptance 9: the speed-up model reproduces its analytic limits
    exactly (n p when T_mem = 0; 1 when n p = 1 and T_mem = 0), and the
    regression point of SPEC.md:462 is the formula's value."""
    from paper_1301_4195_b200.solver import predict_speedup
    assert predict_speedup(4, 16, 16, 256, 0.0, 1e-9, 10.0) == 64.0
    assert predict_speedup(1, 1, 24, 64, 0.0, 1e-9, 10.0) == 1.0
    v = predict_speedup(2, 16, 24, 64, 100.0, 1.0, 10.0)
    w = 10 * 64 * 24 ** 6
    assert v == w / (4 * 2 * 24 ** 3 * 100.0 + w / 32)
    assert 31.9 < v < 32.0
    with pytest.raises(Exception):
        predict_speedup(0, 16, 24, 64, 1.0, 1.0, 10.0)

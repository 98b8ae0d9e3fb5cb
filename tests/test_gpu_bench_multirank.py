"""bench.py's multi-rank path (what the driver's SCALE run launches), as 2 ranks
folded onto the one visible GPU with BOLTZ_BENCH_DIST=gloo: the timing
collectives run on gloo and the cfg3 halo goes through host memory, so no
kernel of one rank ever waits on the other's.  A plumbing check only -- its
timings are not bench values; the NCCL halo itself needs one GPU per rank."""
import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_bench_two_ranks_gloo_folded_prints_one_line_and_shards_cfg3_bitwise():
    env = dict(os.environ, BOLTZ_BENCH_DIST="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--cells", "1024", "--no-n32", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=540)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["unit"] == "evals/s"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    # per-rank work is fixed (weak scaling): the aggregate counts both ranks' cells
    assert d["config"]["cells_per_gpu"] == 1024
    c3 = d["cfg3"]
    assert "error" not in c3, c3
    assert c3["ranks"] == 2 and c3["scaling"] == "strong"
    assert c3["bitwise_vs_1rank"] is True              # decomposition transparency
    n3 = 16 ** 3
    assert c3["halo_bytes_per_step"]["per_boundary_each_way"] == 4 * 2 * n3 * 8
    assert d["parity"]["max_rel_increment_n16_device"] < 1e-10

"""bench.py's contract on CPU: the reference arm (the oracle port of the
reference's OpenMP collision path) prints one JSON line with the SAME metric
string and config as the GPU arm (the driver divides the two; round 1's lines
differed and the ratio was void), its bounded sample stated, and an e2e object
with zero copies."""
import json
import os
import pathlib
import subprocess
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent


def test_reference_arm_line_matches_gpu_arm_contract():
    sys.path.insert(0, str(REPO))
    import bench
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC
    assert d["config"] == bench.workload_config(bench.CELLS, 1)
    assert d["unit"] == "evals/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] == cb["physical_cores"] >= 1 and cb["cpu_model"]
    assert "OMP_PROC_BIND=close" in cb["omp"] and "16 of the 4096" in d["sample"]


def test_host_cpu_counts_physical_cores():
    sys.path.insert(0, str(REPO))
    import bench
    hw = bench.host_cpu()
    assert 1 <= hw["physical_cores"] <= hw["logical_cpus"]

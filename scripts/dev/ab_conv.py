"""Time the K2 convolution of each library variant (development aid).
    python scripts/dev/ab_conv.py variants/lib_*.so
Each variant runs in its own process (BOLTZ_LIB_VARIANT)."""
import os, pathlib, subprocess, sys, json
ROOT = pathlib.Path(__file__).resolve().parents[2]
if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        env = dict(os.environ, BOLTZ_LIB_VARIANT=str(pathlib.Path(lib).resolve()))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(pathlib.Path(lib).name, r.stdout.strip() or r.stderr[-800:], flush=True)
    sys.exit(0)
sys.path.insert(0, str(ROOT))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
out = {}
for n, L, cells in [(16, 6.0, 4096), (32, 8.0, 1024), (24, 8.0, 1024)]:
    if os.environ.get("AB_ONLY16") and n != 16:
        continue
    grid = VelocityGrid.create(n, L)
    op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
    f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
    fh = op.forward(f)
    op.evaluate_qhat(fh)
    op.timing(reset=True); op.set_timing(True)
    for _ in range(3):
        op.evaluate_qhat(fh)
    ms, cnt = op.timing(reset=True)
    t = ms["conv"] / 3  # per evaluate_qhat (a conv may be several kernels: k-chunks, segments)
    out[n] = round(10 * 27 / 64 * n ** 6 * cells / (t * 1e-3) / 1e12, 2)
    op.close()
print(json.dumps({"conv_TFLOPs_alg": out}))

"""N=32 collide timing (mirror path, k_conv_kcsr included) for the library in BOLTZ_LIB_VARIANT (dev aid)."""
import sys, json
sys.path.insert(0, '.')
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
n, L, cells = 32, 8.0, int(sys.argv[1]) if len(sys.argv) > 1 else 1024
grid = VelocityGrid.create(n, L)
G = generate_table(grid, KernelSpec(1.0))
op = CollisionOperator(grid, KernelSpec(1.0), G); del G
f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
q = op.collide(f)
op.timing(reset=True); op.set_timing(True)
for _ in range(3): q = op.collide(f)
ms, cnt = op.timing(reset=True)
print(json.dumps({"conv_ms_per_call": round(ms["conv"] / 3, 2), "evals_s": round(cells * 3 / (sum(ms.values()) * 1e-3)), "sum": float(q.abs().sum())}))

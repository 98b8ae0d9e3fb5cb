#!/bin/bash
# N=32 conv A/B (dev aid): only the 32 entry of ab_conv
for v in "$@"; do
  echo -n "$(basename $v) "
  BOLTZ_LIB_VARIANT=$PWD/$v python - <<'PY'
import sys, json, pathlib
sys.path.insert(0, '.')
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
n, L, cells = 32, 8.0, 1024
grid = VelocityGrid.create(n, L)
G = generate_table(grid, KernelSpec(1.0))
op = CollisionOperator(grid, KernelSpec(1.0), G); del G
f = torch.from_numpy(scenarios.mixture_cells(grid, cells, seed=1)).cuda()
fh = op.forward(f); op.evaluate_qhat(fh)
op.timing(reset=True); op.set_timing(True)
for _ in range(2): op.evaluate_qhat(fh)
ms, cnt = op.timing(reset=True)
print(json.dumps({"n32_TFLOPs_alg": round(10*27/64*n**6*cells*2/(ms["conv"]*1e-3)/1e12, 2)}))
PY
done

# K2 joint longest-first tail (BOLTZ_LPT_TAIL) sweep on cfg2: device value and pinned/pageable e2e
for t in ${TAILS:-1 2 3 4 6}; do
  for rep in 1 2; do
    BOLTZ_LPT_TAIL=$t python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tail $t', round(d['value']), round(d['e2e']['value']), round(d['e2e_pageable']['value']), round(d['kernel_ms']['conv']/d['kernel_launches']['conv'],4), flush=True)"
  done
done

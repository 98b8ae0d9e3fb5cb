# bench value / e2e / pageable per library variant (BOLTZ_LIB_VARIANT), alternating
for r in 1 2 3; do for v in "$@"; do
  BOLTZ_LIB_VARIANT=$PWD/variants/lib_$v.so python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']))"
done; done

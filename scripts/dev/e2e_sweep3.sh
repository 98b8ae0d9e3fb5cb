# e2e pinned / pageable across host chunk schedules with 128-cell edge chunks (current build)
run() { env "$@" python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']))"; }
for r in 1 2; do
for ch in 1,2,3,5,5,3,2,1 1,2,4,6,6,6,4,2,1 1,3,6,6,6,6,3,1 1,2,4,8,8,4,2,1 1,3,8,8,8,3,1 1,2,3,4,6,6,4,3,2,1; do run BOLTZ_HOST_CHUNKS=$ch; done
done

# e2e (pinned and pageable) across host-pipeline chunk schedules (BOLTZ_HOST_CHUNKS)
run() { env "$@" python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']),round(d['e2e_pageable']['ratio_to_pinned'],3))"; }
for ch in 1,2,4,4,2,1 0.5,2,4,4,2,0.5 0.5,1.5,4,4,1.5,0.5 1,2,5,5,2,1 0.5,2,5,5,2,0.5 1,3,5,5,3,1 0.5,1,2,4,4,2,1,0.5 1,2,6,6,2,1; do
run BOLTZ_HOST_CHUNKS=$ch
done

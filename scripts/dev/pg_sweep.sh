# pageable-vs-pinned e2e sweep (defaults: 12 copy threads, streaming stores, 4 MiB blocks, chunks 1,2,4,4,2,1)
run() { env "$@" python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']),round(d['e2e_pageable']['ratio_to_pinned'],3))"; }
run X=1; run X=2; run X=3
run BOLTZ_BOUNCE_BLK_MB=8
run BOLTZ_HOST_CHUNKS=1,2,5,5,2,1
run BOLTZ_HOST_CHUNKS=1,3,4,4,3,1
run BOLTZ_HOST_CHUNKS=1,2,3,4,3,2,1

# copy-thread / block-size sweep of the pageable bounce path with the persistent host threads
run() { env "$@" python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']),round(d['e2e_pageable']['ratio_to_pinned'],3))"; }
run BOLTZ_COPY_THREADS=4; run BOLTZ_COPY_THREADS=6; run BOLTZ_COPY_THREADS=8; run BOLTZ_COPY_THREADS=12; run BOLTZ_COPY_THREADS=16
run BOLTZ_BOUNCE_BLK_MB=1; run BOLTZ_BOUNCE_BLK_MB=2; run BOLTZ_BOUNCE_BLK_MB=8
run BOLTZ_COPY_THREADS=8 BOLTZ_BOUNCE_BLK_MB=2
run BOLTZ_HOST_CHUNKS=1,2,4,4,2,1; run BOLTZ_HOST_CHUNKS=0.5,1,2,3,5,5,3,2,1,0.5

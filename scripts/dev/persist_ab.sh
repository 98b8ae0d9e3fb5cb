# persistent bounce-pipeline host threads (BOLTZ_BOUNCE_PERSIST, default 1) against per-call std::threads
run() { env "$@" python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']),round(d['e2e_pageable']['ratio_to_pinned'],3))"; }
run BOLTZ_BOUNCE_PERSIST=0; run BOLTZ_BOUNCE_PERSIST=1; run BOLTZ_BOUNCE_PERSIST=0; run BOLTZ_BOUNCE_PERSIST=1

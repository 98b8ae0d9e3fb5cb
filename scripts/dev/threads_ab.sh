# default copy team (6 threads) against 12, two runs each, persistent pipeline threads
run() { env "$@" python bench.py --steps 20 --warmup 5 --no-n32 --no-cfg3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*',round(d['value']),round(d['e2e']['value']),round(d['e2e_pageable']['value']),round(d['e2e_pageable']['ratio_to_pinned'],3))"; }
run X=default; run BOLTZ_COPY_THREADS=12; run X=default; run BOLTZ_COPY_THREADS=12; run BOLTZ_COPY_THREADS=4; run BOLTZ_COPY_THREADS=4

#!/bin/bash
run() { echo "== $*"; env "$@" timeout 300 python bench.py --config ${CFG:-c3} --steps 5 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['roofline']['pass_ms'], d['config']['plan'][1][-50:])
    else: print(l[:200])
"; }
EFFT_C64_TILE=3 timeout 200 python tools/gpu_check.py 1048576,2097152,4194304,16777216 2>&1 | cut -c 1-70
run EFFT_C64_TILE=512
run EFFT_C64_TILE=3
CFG=c2 run EFFT_C64_TILE=512
CFG=c2 run EFFT_C64_TILE=3

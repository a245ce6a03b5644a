#!/bin/bash
run() { echo "== $*"; env "$@" timeout 300 python bench.py --config c3 --steps 5 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['roofline']['pass_ms'], d['config']['plan'][1][-70:])
    else: print(l[:200])
"; }
run EFFT_C64_TILE=512
run EFFT_C64_TILE=512 EFFT_DIAG_NOWAIT=2
run EFFT_C64_TILE=512 EFFT_DIAG_NOWAIT=3
run EFFT_C64_TILE=1
run EFFT_C64_TILE=256 EFFT_DIAG_NOWAIT=3
run EFFT_WS=1 EFFT_DIAG_NOWAIT=1

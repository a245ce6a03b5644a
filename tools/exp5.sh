#!/bin/bash
run() { echo "== $*"; env "$@" timeout 300 python bench.py --config c3 --steps 5 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['roofline']['pass_ms'])
    else: print(l[:200])
"; }
run EFFT_DIAG_NOWAIT=0
run EFFT_DIAG_NOWAIT=3
run EFFT_DIAG_NOWAIT=7
run EFFT_DIAG_NOWAIT=15
run EFFT_DIAG_NOWAIT=12
run EFFT_DIAG_NOWAIT=4

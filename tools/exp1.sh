#!/bin/bash
# scheduling experiments on C3 (dev tool)
run() { echo "== $*"; env "$@" timeout 300 python bench.py --config c3 --steps 5 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['roofline']['pass_ms'], d['config']['plan'][1][-40:])
    else: print(l[:200])
"; }
run EFFT_WS=0
run EFFT_WS=0 EFFT_DIAG_NOWAIT=1
run EFFT_WS=0 EFFT_LAG=8 EFFT_SLOTS=16
run EFFT_WS=0 EFFT_LAG=2 EFFT_SLOTS=12
run EFFT_WS=1
run EFFT_WS=1 EFFT_DIAG_NOWAIT=1
run EFFT_WS=1 EFFT_LAG=10 EFFT_SLOTS=20

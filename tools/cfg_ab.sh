#!/bin/bash
# dev: A/B of an env setting over the bench configs (device-timed only)
for c in ${CONFIGS:-c3 c2 c4 r27 r30}; do
  for v in ${VALS:-0 1}; do
    export ${VAR:-EFFT_LEAN_LAGPLUS}=$v
    timeout -s KILL 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-parity 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '$v', d['ms_per_step'], d['roofline']['pass_ms'], [p.split('lag=')[1] for p in d['config']['plan'] if 'lag=' in p])"
  done
done

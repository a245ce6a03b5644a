#!/bin/bash
# dev: lag / slot sweep of the shipping paired kernel at 2^30 (both passes paired: EFFT_LEAN_WIDE=0)
export EFFT_LEAN_WIDE=${WIDE:-0}
for ls in ${LS:-8:13 9:14 10:15 10:16 11:16 11:18 12:18 13:20 14:22}; do
  echo -n "lag ${ls%%:*} slots ${ls##*:}: "
  EFFT_LEAN_LAG=${ls%%:*} EFFT_LEAN_SLOTS=${ls##*:} timeout -s KILL 120 python tools/pipe_check.py 30 0 10 2>&1 | grep "ms " | sed 's/.*passes//'
done

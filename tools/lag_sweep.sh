#!/bin/bash
# dev: lag / slot sweep of the pipelined kernel at 2^30 (LS="lag:slots ...")
export EFFT_LEAN_PIPE=3
for ls in ${LS:-6:8 8:10 8:12 10:14 12:16} ; do
  echo "== LAG ${ls%%:*} SLOTS ${ls##*:}"
  EFFT_LEAN_LAG=${ls%%:*} EFFT_LEAN_SLOTS=${ls##*:} timeout -s KILL 120 python tools/pipe_check.py 30 3 5 2>&1 | grep "ms "
done

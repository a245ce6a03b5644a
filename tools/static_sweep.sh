#!/bin/bash
# dev: static schedule in the default lean kernels, lag/slots sweep at 2^30
for cfg in ${CFGS:-0:0:0 1:0:0 1:4:8 1:5:9 1:6:10 1:8:12 0:6:10 0:8:12}; do
  IFS=: read st lag sl <<< "$cfg"
  echo "== static $st lag $lag slots $sl"
  if [ "$lag" = 0 ]; then
    EFFT_LEAN_STATIC=$st timeout -s KILL 120 python tools/pipe_check.py 30 0 5 2>&1 | grep -E "ms |lag="
  else
    EFFT_LEAN_STATIC=$st EFFT_LEAN_LAG=$lag EFFT_LEAN_SLOTS=$sl timeout -s KILL 120 python tools/pipe_check.py 30 0 5 2>&1 | grep -E "ms "
  fi
done

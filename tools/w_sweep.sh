#!/bin/bash
export EFFT_LEAN_PIPE=3
for w in ${WS:-1 2 4}; do
  echo "== W $w"
  EFFT_LEAN_W=$w timeout -s KILL 120 python tools/pipe_check.py 30 3 5 2>&1 | grep -E "ms |rel-L2"
done

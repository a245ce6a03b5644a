#!/bin/bash
export EFFT_LEAN_PIPE=3 EFFT_LEAN_LAG=8 EFFT_LEAN_SLOTS=14
for ns in ${NS:-1 32 64 128 256 512}; do
  echo "== nanosleep $ns"
  EFFT_PIPE_ABL=$((ns << 16)) timeout -s KILL 120 python tools/pipe_check.py 30 3 5 2>&1 | grep -E "ms "
done

#!/bin/bash
# dev: ablation sweep of the pipelined kernel at 2^30 (timing only)
export EFFT_LEAN_PIPE=3
for abl in ${ABLS:-0 1 2 3 7 8 15} ; do
  echo "== ABL $abl"
  EFFT_PIPE_ABL=$abl timeout -s KILL 120 python tools/pipe_check.py 30 3 5 2>&1 | grep "ms "
done

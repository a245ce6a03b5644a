#!/bin/bash
# dev: A/B of two builds of the library at 2^28 / 2^30 (alternating, same box)
for rep in 1 2 3; do
  for lib in tools/ab/lib_head.so ""; do
    echo -n "lib=${lib:-current} "
    EFFT_LIB=$lib timeout -s KILL 120 python tools/pipe_check.py ${SIZES:-30} 0 10 2>&1 | grep "ms " | sed 's/.*EFFT_LEAN_PIPE=0://' | tr '\n' ' '
    echo
  done
done

#!/bin/bash
# Sweep the generic two-pass split (EFFT_SPLIT_T1 = log2 of pass-1 radix) on
# the small configs that do not take the lean kernels.
mkdir -p gpurun_out
for t1 in default 8 9 10 11 12 13; do
  if [ "$t1" = default ]; then unset EFFT_SPLIT_T1; else export EFFT_SPLIT_T1=$t1; fi
  echo "== c1 t1=$t1"
  timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], d['value'], d['config']['plan'][1:], d['roofline']['pass_ms'])"
done

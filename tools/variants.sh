#!/bin/bash
# Correctness sweep + timing of the kernel variants (dev tool).
set -u
timeout 300 python tools/gpu_check.py > gpurun_out/checkV.log 2>&1
EFFT_WS=1 timeout 300 python tools/gpu_check.py 1048576,2097152,3145728,4194304 >> gpurun_out/checkV.log 2>&1
python - <<PY
import re
L=open("gpurun_out/checkV.log").read().splitlines()
bad=[l for l in L if "FAIL" in l or (re.search(r"fwd_err=([0-9.e+-]+)",l) and float(re.search(r"fwd_err=([0-9.e+-]+)",l).group(1))>1e-5)]
print("check lines", len(L), "BAD", len(bad)); print("\n".join(x[:200] for x in bad[:10]))
PY
: > gpurun_out/benchV.log
for ws in 0 1; do for c in c3 c1 c2 c4; do
  EFFT_WS=$ws timeout 300 python bench.py --config $c --steps 5 --no-cpu --no-e2e >> gpurun_out/benchV.log 2>&1
done; done
python - <<PY
import json
for l in open("gpurun_out/benchV.log"):
    if l.startswith("{"):
        d=json.loads(l); print(d["config"]["workload"][:40], d["value"], d["ms_per_step"], d["roofline"]["pass_ms"], d["roofline"]["frac"], d["config"]["plan"][1][:50])
    else: print(l[:200])
PY

#!/bin/bash
# GPU-box sanity check (dev tool): smoke, gpu tests, bench lines (C3 + a few others).
set -u
mkdir -p gpurun_out
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
for c in ${CONFIGS:-c2 r30}; do timeout -s KILL 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1; done
tail -n 3 gpurun_out/smoke.log
tail -n 5 gpurun_out/pytest_gpu.log

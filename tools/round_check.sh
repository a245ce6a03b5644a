#!/bin/bash
# GPU-box check: gpu tests, bench (c3), launch list.  Dev tool.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3.log
for c in c2 c4; do timeout 300 python bench.py --config $c --steps 5 --no-cpu --no-e2e >> gpurun_out/bench_other.log 2>&1; done

#!/bin/bash
# GPU-box round check (dev tool): smoke, gpu tests, bench lines for every config,
# launch list + one full ncu capture of the C3 kernels.
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3.log
: > gpurun_out/bench_other.log
for c in c1 c2 c4 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu >> gpurun_out/bench_other.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/prof_run.py c3 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lean -c 2 -o gpurun_out/lean_c3 \
    python tools/prof_run.py c3 1 > gpurun_out/ncu_full.log 2>&1
echo done

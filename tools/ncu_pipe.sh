#!/bin/bash
# dev: full ncu capture of the pipelined kernel at 2^30 (both passes, one launch each)
export EFFT_LEAN_PIPE=${EFFT_LEAN_PIPE:-3}
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:lean_ -s 2 -c 2 -f -o gpurun_out/pipe_c3 \
  python tools/prof_run.py c3 2 > gpurun_out/ncu_pipe.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/pipe_c3.ncu-rep > gpurun_out/pipe_c3_summary.txt 2>&1
tail -n 5 gpurun_out/ncu_pipe.log

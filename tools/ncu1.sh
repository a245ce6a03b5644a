set -u
python tools/prof_run.py c3 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:staged_kernel -c 1 -o gpurun_out/ws_cur python tools/prof_run.py c3 1 > gpurun_out/ncu1.log 2>&1
echo rc=$?

python tools/prof_run.py c3 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lean_pair -c 2 -o gpurun_out/lean_pair python tools/prof_run.py c3 1 > gpurun_out/ncu_pair.log 2>&1

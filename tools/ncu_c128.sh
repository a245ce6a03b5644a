# ncu captures of the complex128 lean kernels (C2 and C4 shapes), one pass each
python tools/prof_run.py c2 1 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none -k regex:lean -c 2 -o gpurun_out/lean_c2 python tools/prof_run.py c2 1 > gpurun_out/ncu_c2.log 2>&1
python tools/prof_run.py c4 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none -k regex:lean -c 2 -o gpurun_out/lean_c4 python tools/prof_run.py c4 1 > gpurun_out/ncu_c4.log 2>&1
echo done

set -u
python tools/prof_run.py c3 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lean -c 1 -o gpurun_out/lean_reg python tools/prof_run.py c3 1 > gpurun_out/ncu_lean.log 2>&1
EFFT_LEAN_DIAG=1 ncu --set full --clock-control none -k regex:lean -c 1 -o gpurun_out/lean_diag python tools/prof_run.py c3 1 >> gpurun_out/ncu_lean.log 2>&1
echo rc=$?

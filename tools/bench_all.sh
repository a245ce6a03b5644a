#!/bin/bash
# Every config through bench.py (our arm + the reference arm), then the C3 ncu
# launch list and one full capture of the dominant C3 pass kernel.
# Usage (on the GPU box): bash tools/bench_all.sh <tag>
tag=${1:-sweep}
out=gpurun_out/$tag
mkdir -p $out
for c in c3 c1 c2 c4 r24 r27 r30 c5; do
  steps=20; [ $c = c5 ] && steps=5
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
  echo "$c rc=$?"
  rs=5; [ $c = c5 ] && rs=1; [ $c = c4 ] && rs=2
  timeout 900 python bench.py --config $c --impl reference --steps $rs --warmup 1 > $out/ref_$c.json 2> $out/ref_$c.err
  echo "ref $c rc=$?"
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
# launch list (serialised, cold): shares only
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $out/c3_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:lean_ -s 2 -c 2 -o $out/c3_full \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $out/ncu_full.log 2>&1
echo "ncu full rc=$?"

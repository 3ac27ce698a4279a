#!/bin/bash
# Round-1 evidence refresh on one B200: bench lines for every config, the reference arm, the
# ncu launch list of the default bench command and a full ncu capture of the top kernel.
set -u
O=gpurun_out/r01
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > $O/smi.txt
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err
echo "ref rc=$?" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/ncu_launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch_run.log 2>&1
echo "ncu launches rc=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_cluster -c 1 -o $O/ncu_jacobi_c2 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_run.log 2>&1
echo "ncu full rc=$?" >> $O/status.txt

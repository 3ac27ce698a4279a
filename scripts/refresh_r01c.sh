#!/bin/bash
set -u
O=gpurun_out/r01c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > $O/smi.txt
./scripts/chol_probe 272 > $O/chol_trace_272.txt 2>&1
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?" >> $O/status.txt
done
bash scripts/ncu_launches.sh $O >> $O/status.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_tiles_kernel -s 2 -c 1 \
  -o $O/ncu_chol_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_chol.log 2>&1
echo "ncu chol rc=$?" >> $O/status.txt

#!/bin/bash
# ncu launch list of our kernels in the default bench command (input synthesis excluded)
O=${1:-gpurun_out/r01}
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k 'regex:lramm::' -c 500 --csv --log-file $O/ncu_launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch_run.log 2>&1
echo "ncu launches rc=$?"

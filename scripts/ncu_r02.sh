#!/bin/bash
# Round-2 evidence: (1) ncu launch list of the default (c3) bench command, our kernels only;
# (2) one full capture of the dominant kernel (the tridiagonalisation, c3 shape) and of the c3
# sketch GEMM.  Each only after the same command has exited 0 without ncu.
O=${1:-gpurun_out/r02}
mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k 'regex:lramm::' -c 1200 --csv --log-file $O/ncu_launches_c3.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy > $O/ncu_launch_run.log 2>&1
echo "ncu launches rc=$?"
EIG_REPS=1 timeout 300 python scripts/eig_check.py 544 > $O/plain_eig.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sytrd_push_kernel -s 1 -c 1 \
  -o $O/ncu_sytrd_c3 -f env EIG_REPS=1 python scripts/eig_check.py 544 > $O/ncu_sytrd.log 2>&1
echo "sytrd rc=$?"

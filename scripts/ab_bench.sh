#!/usr/bin/env bash
# A/B of environment switches on one bench config: scripts/ab_bench.sh c3 "X=1" "LRAMM_TRSM_INV=1" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfg=$1; shift
: > gpurun_out/ab_summary.txt
for e in "$@"; do
  env $e timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/ab.log 2>&1
  rc=$?
  r=$(grep '^{' gpurun_out/ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1))' 2>/dev/null)
  echo "$cfg $e rc=$rc $r" >> gpurun_out/ab_summary.txt
done
cat gpurun_out/ab_summary.txt

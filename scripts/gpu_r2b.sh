#!/usr/bin/env bash
# c3 default bench (pipelined e2e) + c4 with several graph / stream splits
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "c3 rc=$?"
for gs in "1 8" "4 8" "8 8" "8 16" "16 32" "1 32"; do
  set -- $gs
  BENCH_GRAPHS=$1 BENCH_STREAMS=$2 timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c4_g$1_s$2.log 2>&1
  echo "c4 graphs=$1 streams=$2 rc=$?"; python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c4_g$1_s$2.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"])
PY
done

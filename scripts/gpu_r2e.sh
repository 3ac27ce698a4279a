#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/e2e_timeline.py 3 4 > gpurun_out/e2e_timeline_3.txt 2>&1; grep -v sytrd gpurun_out/e2e_timeline_3.txt | tail -60
for inf in 2 3 4; do
  BENCH_E2E_INFLIGHT=$inf timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3_inf$inf.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3_inf$inf.log").read().strip().splitlines()[-1])
print($inf, d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"))
if $inf == 3:
    for k in d["top_kernels"]: print("   ", k)
PY
done

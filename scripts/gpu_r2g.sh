#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/e2e_timeline.py 4 5 > gpurun_out/e2e_timeline_4.txt 2>&1; grep -v "Warn\|warn" gpurun_out/e2e_timeline_4.txt | grep "per call\|host thread\|union" | tail -30
for cfgs in "1 2" "1 3" "1 4" "1 6" "2 4"; do
  set -- $cfgs
  LRAMM_HOST_COMPUTE_SLOTS=$1 BENCH_E2E_INFLIGHT=$2 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3_s$1_inf$2.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3_s$1_inf$2.log").read().strip().splitlines()[-1])
print("slots $1 inflight $2:", d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"))
PY
done

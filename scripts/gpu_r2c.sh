#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/pcie_probe.py 2>&1 | tee gpurun_out/pcie_probe.txt
for inf in 1 2 3 4; do
  BENCH_E2E_INFLIGHT=$inf timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3_inf$inf.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3_inf$inf.log").read().strip().splitlines()[-1])
print($inf, d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"))
PY
done

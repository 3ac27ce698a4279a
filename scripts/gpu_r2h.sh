#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_concurrency.py -m gpu -q -x > gpurun_out/pytest_conc.log 2>&1; tail -15 gpurun_out/pytest_conc.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; tail -5 gpurun_out/pytest.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c4.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c4.log").read().strip().splitlines()[-1])
print("c4", d["ms_per_step"], d["value"], d["e2e"])
PY

#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/eig_check.py > gpurun_out/eig_pre.log 2>&1; echo "eig rc=$?"; tail -25 gpurun_out/eig_pre.log
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/pytest_part.log 2>&1; tail -3 gpurun_out/pytest_part.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3.log").read().strip().splitlines()[-1])
print("c3", d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"))
for k in d["top_kernels"][:8]: print("   ", k)
print(d["roofline"]["kernel"], d["roofline"]["frac"])
PY

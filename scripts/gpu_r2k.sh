#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for args in "8192 544 8192 f64" "8192 544 8192 f64 row" "4096 272 4096 f64 row" "8192 8192 512 f32"; do
  python scripts/igemm_once.py $args 2>&1 | tail -1
done
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_configs.py tests/test_gpu_edge_shapes.py -m gpu -q -x > gpurun_out/pytest_part.log 2>&1; tail -3 gpurun_out/pytest_part.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3.log").read().strip().splitlines()[-1])
print("c3", d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"))
for k in d["top_kernels"][:8]: print("   ", k)
PY

#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/qr_prof.py 8192 544 2>&1 | grep "qr 8192\|trinv\|chol_tiles\|kernel sum"
python scripts/qr_prof.py 131072 1056 2>&1 | grep "qr 1310\|trinv\|chol_tiles\|kernel sum"
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "qr" > gpurun_out/pytest_qr.log 2>&1; tail -3 gpurun_out/pytest_qr.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3.log").read().strip().splitlines()[-1])
print("c3", d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"))
print(d["accuracy"]["fast_mode_rel_diff_vs_restatement"])
for k in d["top_kernels"][:6]: print("   ", k)
PY

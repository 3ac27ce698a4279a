#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3.log").read().strip().splitlines()[-1])
print("c3", d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"], d["e2e"].get("single_call_ms"), d["gpu_launches_per_step"])
print(d["accuracy"])
for k in d["top_kernels"][:8]: print("   ", k)
PY
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; tail -5 gpurun_out/pytest.log
for c in c2 c1 c5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['accuracy'].get('fast_mode_rel_diff_vs_restatement'), d['accuracy'].get('rel_err_vs_exact'), d['accuracy'].get('reference_rel_err_vs_exact'))"; done

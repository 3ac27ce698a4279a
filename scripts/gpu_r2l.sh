#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c3 c4 c2 c1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_$c.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$c.log").read().strip().splitlines()[-1])
print("$c", round(d["ms_per_step"],3), round(d["value"],2), "e2e", round(d["e2e"]["ms_per_step"],2), d["e2e"].get("single_call_ms"))
PY
done
BENCH_STREAMS=32 timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 s32', d['ms_per_step'], d['e2e']['ms_per_step'])"

#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in default 8; do
  if [ "$r" = default ]; then unset LRAMM_TRSM_INV_RATIO; else export LRAMM_TRSM_INV_RATIO=$r; fi
  timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-accuracy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 ratio $r', d['ms_per_step'], d['value'])"
done
unset LRAMM_TRSM_INV_RATIO
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c5.log 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_c5.log').read().strip().splitlines()[-1]); print('c5', d['ms_per_step'], d['value'], d['e2e']['ms_per_step'])
for k in d['top_kernels'][:8]: print('   ', k)"

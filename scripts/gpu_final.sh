#!/usr/bin/env bash
# What the driver runs at round end: GPU tests, smoke, the default bench and the reference arm.
cd "$(dirname "$0")/.."
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?"
timeout 1200 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
python - <<PY
import json
for c in ("c3", "c4"):
    d=json.loads(open("$O/bench_%s.json" % c).read().strip().splitlines()[-1])
    print(c, round(d["ms_per_step"],3), round(d["value"],2), "e2e", round(d["e2e"]["ms_per_step"],2), d["e2e"].get("single_call_ms"), d.get("cpu_baseline",{}).get("value"), d["roofline"]["frac"], d["clocks"])
PY

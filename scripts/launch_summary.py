"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/launch_summary.py gpurun_out/launches_c2.csv [first_kernel_regex]

Lists every launch's kernel and duration, then per-kernel totals for one lramm step: the
launches from the N-th occurrence of the step's first kernel (default: the sketch quantiser
`absmax_tile_kernel`, second step) up to the next occurrence.
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
first = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"absmax_tile_kernel")
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
launches = []
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    us = v / 1e3 if unit == "nsecond" else (v * 1e3 if unit == "msecond" else v if unit == "usecond" else v / 1e3)
    name = r["Kernel Name"].replace("lramm::(anonymous namespace)::", "").replace("void ", "")
    launches.append((name.split("(")[0], us))
starts = [i for i, (n, _) in enumerate(launches) if first.search(n)]
# steps issue A and B sketches back to back: a step begins at every other match
steps = starts[::2]
if len(steps) >= 3:
    lo, hi = steps[1], steps[2]
elif len(steps) >= 2:
    lo, hi = steps[0], steps[1]
else:
    lo, hi = 0, len(launches)
agg = collections.defaultdict(lambda: [0.0, 0])
for n, us in launches[lo:hi]:
    agg[n][0] += us
    agg[n][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"{len(launches)} launches captured; one step = launches [{lo}, {hi}) = {hi - lo} launches, "
      f"serialised sum {tot / 1e3:.3f} ms (cold-cache, one kernel at a time)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{v[0]:10.1f} us {100 * v[0] / tot:5.1f}%  {v[1]:4d}x  {k}")

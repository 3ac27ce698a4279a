"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals (optionally last fraction)."""
import csv, collections, sys
path = sys.argv[1]; frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
data = data[int(len(data) * (1 - frac)):]
agg = collections.OrderedDict(); cnt = collections.Counter(); tot = 0.0
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in data:
    name = r[ki].split("(")[0].replace("lramm::<unnamed>::", "")[:60]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
    agg[name] = agg.get(name, 0) + v; cnt[name] += 1; tot += v
print(f"{'us':>10} {'n':>5} {'us/launch':>10}  kernel   (total {tot:.1f} us, {sum(cnt.values())} launches)")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} {cnt[k]:5d} {v / cnt[k]:10.2f}  {k}")

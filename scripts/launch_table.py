"""Print an ncu --metrics gpu__time_duration.sum CSV launch list as 'id  kernel  us'."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = 0.0
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        us = float(d["Metric Value"].replace(",", "")) / 1e3
        tot += us
        print(f"{d['ID']:>4} {d['Kernel Name'][:70]:70s} {us:9.1f}")
print(f"total {tot:.1f} us")

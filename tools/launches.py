"""Summarise an ncu launch list (gpu__time_duration per kernel launch)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")[:70]
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1000.0)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>5s} {'mean_us':>10s} {'min_us':>10s} {'share':>7s}")
for k, v in agg.items():
    print(f"{k:70s} {len(v):5d} {sum(v)/len(v):10.1f} {min(v):10.1f} {sum(v)/tot:7.1%}")

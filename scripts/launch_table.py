"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, data = rows[0], rows[1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name")
data = [r for r in data if r[mi] == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in data:
    name = r[ki].split("(")[0].split("<")[0][-40:]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale
tot = sum(a[1] for a in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:42s} {c:6d} {t:12.1f} us {100 * t / tot:5.1f}%")
print(f"total {tot:.1f} us")

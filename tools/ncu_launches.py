"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel (time share)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= max(ki, vi, ui):
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").strip()[:70]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'us total':>10} {'launches':>8} {'us/launch':>10} {'share':>6}  kernel")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} {c:8d} {t / c:10.1f} {100 * t / tot:5.1f}%  {k}")
print(f"{tot:10.1f} total us")

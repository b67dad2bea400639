"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ui, vi = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")[:70]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {t:10.3f} {100 * t / tot:6.2f}%  {k}")

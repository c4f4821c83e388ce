"""Mean per-kernel duration from an ncu launch-list CSV (gpu__time_duration.sum): python scripts/launch_summary.py F"""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    agg.setdefault(r[ki][:80], []).append(float(r[vi].replace(",", "")))
for n, v in agg.items():
    print(f"{len(v):4d} {sum(v) / len(v) / 1e3:9.1f} us  {n}")

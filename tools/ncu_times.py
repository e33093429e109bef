"""Average per-launch time by kernel from a tools/ncu_times.sh CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if "Kernel Name" in r)
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
t = collections.defaultdict(list)
for r in rows[rows.index(h) + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        t[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v) / 1e3:9.2f} ms  n={len(v):4d}  avg={sum(v) / len(v):8.1f}  {k}")

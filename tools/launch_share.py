"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: share of device time per kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"])
    name = re.sub(r"sb::|<unnamed>::|\(anonymous namespace\)::", "", name)[:80]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "nsecond")
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(unit, 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'share':>7} {'launches':>8} {'avg us':>10}  kernel   (total {tot / 1e3:.1f} ms over {sum(v[0] for v in agg.values())} launches)")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t / tot * 100:6.2f}% {n:8d} {t / n:10.1f}  {k}")

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (ms)."""
import collections
import csv
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
d = collections.defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
        d[r["Kernel Name"][:70]].append(float(r["Metric Value"].replace(",", "")) * scale)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v):9.3f} ms  total={sum(v):9.2f} ms  {100*sum(v)/tot:5.1f}%")

"""Per-source-line warp-stall samples from `ncu -i REP --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
f = None
agg = {}
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0].isdigit() and len(r) > 4 and r[4].isdigit():
        agg[(f, int(r[0]))] = (int(r[4]), r[1])
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for (f, l), (v, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{f}:{l} {v} {100 * v / tot:.1f}%  {s.strip()[:90]}")

"""Per-sweep kernel composition from an ncu launch list of tools/sweep_launches.py (NVTX ranges
"ascent" and "hals", 3 sweeps each): mean ms per sweep per kernel and its share of the sweep.
    python tools/sweep_summary.py gpurun_out/x_sweep_launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
col = [k for k in rows[0] if k.startswith("thread Domain:Push/Pop")][0]
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
groups = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    stage = "ascent" if "ascent" in r[col] else ("hals" if "hals" in r[col] else "?")
    name = r["Kernel Name"].split("(")[0][:60]
    groups[stage][name].append(float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-6))
for stage, d in groups.items():
    tot = sum(sum(v) for v in d.values()) / 3
    print(f"== {stage}: {tot:.3f} ms per sweep (kernel time, serialised, cold-ish caches), "
          f"{sum(len(v) for v in d.values()) / 3:.0f} launches per sweep")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:60s} {sum(v) / 3:8.3f} ms  {100 * sum(v) / 3 / tot:5.1f} %  x{len(v) // 3}")

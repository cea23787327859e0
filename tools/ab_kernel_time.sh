# per-launch device time of one kernel (regex $1) for ab_old/ vs the current tree
K=${1:-tc_pbcd_kernel}
for v in old new; do
  if [ $v = old ]; then b=ab_old/bench.py; else b=bench.py; fi
  timeout 600 ncu -k regex:$K --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt_$v.csv python $b --steps ${2:-6} --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python - $v <<'PY'
import csv, sys
rows=[r for r in csv.DictReader(l for l in open(f'gpurun_out/kt_{sys.argv[1]}.csv') if l.startswith('"')) if r["Metric Name"]=="gpu__time_duration.sum"]
x=[float(r["Metric Value"].replace(',',''))*(1e-3 if r["Metric Unit"]=="ns" else 1) for r in rows]
x=[a for a in x if a > 20]
print(sys.argv[1], len(x), 'us', [round(a) for a in x[:10]])
PY
done

# tensor-core HALS check: parity tests with ENMF_TC_HALS=1, then an alternating bench A/B
mkdir -p gpurun_out
ENMF_TC_HALS=1 timeout 900 python -m pytest tests -q -m gpu -x -k "${1:-hals or trajectory or final or edge or fullsize or iterate_host or multirank}" > gpurun_out/hals_tests.log 2>&1
tail -15 gpurun_out/hals_tests.log
for rep in 1 2; do
  for v in 0 1; do
    ENMF_TC_HALS=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hals_tc=$v', round(d['value'],3), {k: round(v,2) for k, v in d['config'].get('stage_rates', {}).items()}, d['clocks']['sm_mhz'])"
  done
done
ENMF_TC_HALS=1 timeout 600 ncu -k regex:hals --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h1.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_ncu1.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/h1.csv') if l.startswith('"')) if r["Metric Name"]=="gpu__time_duration.sum"]
x=[float(r["Metric Value"].replace(',',''))*(1e-3 if r["Metric Unit"]=="ns" else 1) for r in rows]
print('tc_hals us', [round(a) for a in x if a > 20][:8])
PY

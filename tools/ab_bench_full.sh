# A/B of the default bench (100 sweeps) between ab_old/ and the current tree, alternating
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then b=ab_old/bench.py; else b=bench.py; fi
    timeout 600 python $b --no-cpu-baseline --no-e2e --no-ablation 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],3), {k: round(v,2) for k, v in d['config'].get('stage_rates', {}).items()}, d['roofline']['pass_ms'], d['clocks']['sm_mhz'])"
  done
done

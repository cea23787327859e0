# A/B of bench.py numbers: ab_old/ (previous build) vs the current tree, alternating.
# usage: bash tools/ab_bench.sh [bench args]
ARGS=${@:-"--steps 30 --warmup 3 --no-cpu-baseline --no-e2e"}
for rep in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then b=ab_old/bench.py; else b=bench.py; fi
    timeout 600 python $b $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],3), {k: round(v,2) for k, v in d['config'].get('stage_rates', {}).items()}, d['clocks']['sm_mhz'])"
  done
done

# A/B of X-pass variants in one box session: old package (ab_old/), current, current + pair.
mkdir -p gpurun_out; : > gpurun_out/ab.log
for rep in 1 2; do
  for v in old new pair; do
    if [ $v = old ]; then b=ab_old/bench.py; else b=bench.py; fi
    if [ $v = pair ]; then ev=1; else ev=0; fi
    line=$(ENMF_TC_PAIR=$ev timeout 600 python $b --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
    echo "$v $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["pass_ms"], d["clocks"]["sm_mhz"])')" >> gpurun_out/ab.log
  done
done
cat gpurun_out/ab.log

# Round B with classes <= 2, smoke (well-posed ascent part), sparse SVD vs oracle, multirank
# sliced pass 2, C5 sweep times; pair-kernel A/B at the power cap.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-b12}
timeout 600 python tools/kstar_probe.py > gpurun_out/${T}_kstar.log 2>&1; tail -12 gpurun_out/${T}_kstar.log | head -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; tail -2 gpurun_out/${T}_smoke.log
timeout 1800 python -m pytest tests -q -m gpu -x -s -k "(ascent and tc) or stages or fullsize or multirank or sparse or fused" > gpurun_out/${T}_tests.log 2>&1
grep -E "per-update|full size|sparse exact|passed|failed|Error" gpurun_out/${T}_tests.log | head -30
for f in 1 0; do
  ENMF_TC_PAIR=$f timeout 600 python bench.py --no-small --no-ablation --no-cpu-baseline --no-e2e > gpurun_out/${T}_pair$f.log 2>&1
  echo "pair=$f $(tail -1 gpurun_out/${T}_pair$f.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(round(d["value"],2), c["stage_rates"], {k: round(v["ms"],3) for k,v in d["roofline"]["passes"].items()}, d["clocks"]["sm_mhz"])')"
done

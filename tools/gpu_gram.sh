# Tensor-core quantised Gram: parity vs the SIMT Gram, the HALS/trajectory/fullsize tests on
# the tc path, and an A/B of the default bench.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-gr}
timeout 1800 python -m pytest tests -q -m gpu -x -s -k "tc_gram or (hals and tc) or (trajectory and tc) or fullsize or multirank or objective or final" > gpurun_out/${T}_tests.log 2>&1
grep -E "tc Gram|full size|passed|failed|Error" gpurun_out/${T}_tests.log | head -20
for g in 1 0; do
  ENMF_TC_GRAM=$g timeout 900 python bench.py --no-small --no-ablation --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench$g.log 2>&1
  echo "tcgram=$g $(tail -1 gpurun_out/${T}_bench$g.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(round(d["value"],2), c["stage_rates"], {k: round(v["ms"],3) for k,v in d["roofline"]["passes"].items()}, d["clocks"]["sm_mhz"])')"
done

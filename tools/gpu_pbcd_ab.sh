# tc_pbcd_kernel NH = 4 (16 warps) vs NH = 2 (8 warps): parity tests of the ascent on the tensor-
# core path, then alternating bench runs (ascent stage rate).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -s -k "(shadow_ascent and tc) or fullsize or graph_replay or solve_host or fixed_step or (final_objective and tc)" > gpurun_out/ab_tests.log 2>&1
tail -2 gpurun_out/ab_tests.log
for nh in 2 4 2 4; do
  ENMF_TC_PBCD_NH=$nh timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-ablation --no-small > gpurun_out/ab_nh$nh.log 2>&1
  echo "nh=$nh $(tail -1 gpurun_out/ab_nh$nh.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"]["stage_rates"], d["clocks"]["sm_mhz"])')"
done

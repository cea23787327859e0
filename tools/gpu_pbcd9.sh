# tc_pbcd with g's grid integers kept in TMEM class 3: parity (stages bitwise, shadow tc,
# fixed-step ablation, smoke), C5 sweep times, one whole-range U capture.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-b13}
timeout 600 python tools/kstar_probe.py > gpurun_out/${T}_kstar.log 2>&1; sed -n 3,8p gpurun_out/${T}_kstar.log
timeout 1500 python -m pytest tests -q -m gpu -x -s -k "(ascent and tc) or stages or fullsize or fused or ablation or three_ranks or sliced" > gpurun_out/${T}_tests.log 2>&1
grep -E "per-update|full size|fixed-step|passed|failed|Error" gpurun_out/${T}_tests.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; tail -2 gpurun_out/${T}_smoke.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pbcd_kernel -s 32 -c 1 \
    -o gpurun_out/${T}_pbcd python tools/kstar_probe.py > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"

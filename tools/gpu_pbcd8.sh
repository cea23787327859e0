# tc_pbcd_kernel iteration: ascent parity (shadow tc, full size, stages), smoke, C5 sweep
# times, one full ncu capture of a whole-range U launch.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-b9}
timeout 900 python tools/kstar_probe.py > gpurun_out/${T}_kstar.log 2>&1; tail -14 gpurun_out/${T}_kstar.log
timeout 1500 python -m pytest tests -q -m gpu -x -s -k "(ascent and tc) or stages or smoke or fullsize or multirank or sparse or ablation" > gpurun_out/${T}_tests.log 2>&1
grep -E "per-update|full size|passed|failed|Error" gpurun_out/${T}_tests.log | head -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pbcd_kernel -s 32 -c 1 \
    -o gpurun_out/${T}_pbcd python tools/kstar_probe.py > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"

# Full GPU pass on the current tree: parity suite, smoke, default bench, 20-sweep bench,
# launch list of a short bench, full ncu captures of tc_pbcd_kernel (whole-range U launch)
# and tc_hals_kernel (U block, fused).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-rd}
timeout 2400 python -m pytest tests -q -m gpu -rs --durations=10 > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.log 2>&1
tail -1 gpurun_out/${T}_bench20.log | cut -c1-300
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation --no-small"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pbcd_kernel -s 32 -c 1 \
    -o gpurun_out/${T}_pbcd python tools/kstar_probe.py > gpurun_out/${T}_ncu_pbcd.log 2>&1
echo "ncu pbcd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_hals_kernel -s 24 -c 1 \
    -o gpurun_out/${T}_hals python tools/kstar_probe.py > gpurun_out/${T}_ncu_hals.log 2>&1
echo "ncu hals rc=$?"

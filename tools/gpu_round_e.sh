# Final pass of round 2 on the current tree: parity suite, smoke, default bench, launch list of
# a short bench (the same command first without ncu).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-r02e}
timeout 2400 python -m pytest tests -q -m gpu -rs -s --durations=10 > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | cut -c1-400
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation --no-small"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/small_probe.py 200 > gpurun_out/${T}_small.log 2>&1
grep "rep 1" gpurun_out/${T}_small.log
timeout 300 python tools/small_probe.py 4 C3 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_small_launches.csv python tools/small_probe.py 4 C3 > gpurun_out/${T}_ncu_small_launch.log 2>&1
echo "small launch list rc=$?"

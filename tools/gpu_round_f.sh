# Last pass of round 2 on the final tree: parity suite, smoke, default bench, small probe.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-r02f}
timeout 2400 python -m pytest tests -q -m gpu -rs -s --durations=10 > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | cut -c1-400
timeout 300 python tools/small_probe.py 200 > gpurun_out/${T}_small.log 2>&1
grep "rep 1" gpurun_out/${T}_small.log
timeout 300 python tools/init_timing.py > gpurun_out/${T}_init.log 2>&1
tail -12 gpurun_out/${T}_init.log

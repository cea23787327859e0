# Round-2c check of HEAD: GPU parity suite, smoke, default bench.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-rc}
timeout 2400 python -m pytest tests -q -m gpu -rs --durations=15 > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | cut -c1-600

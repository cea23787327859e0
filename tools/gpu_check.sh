# GPU check of the current tree: parity suite, smoke, and a 20-sweep bench.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests -q -m gpu -rs -x --durations=15 > gpurun_out/chk_tests.log 2>&1
tail -25 gpurun_out/chk_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/chk_smoke.log 2>&1
tail -2 gpurun_out/chk_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-ablation > gpurun_out/chk_bench.log 2>&1
tail -1 gpurun_out/chk_bench.log | cut -c1-600

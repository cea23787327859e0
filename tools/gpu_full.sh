# Full GPU check: parity suite, smoke, a 30-step bench and the PBCD launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/b30.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pbcd" --csv --log-file gpurun_out/pbcd_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/b30.log

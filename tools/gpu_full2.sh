# Round-2 GPU pass: parity suite, smoke, default bench, launch list and one full ncu capture
# of the X-pass kernel (each ncu command only after the same command exited 0 without ncu).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests -q -m gpu -rs -s --durations=20 > gpurun_out/r2_tests.log 2>&1
tail -3 gpurun_out/r2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke.log 2>&1
tail -2 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1
tail -1 gpurun_out/r2_bench.log | cut -c1-300
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation"
timeout 600 $CMD > gpurun_out/r2_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_i8_kernel \
    -s 40 -c 2 -o gpurun_out/r2_xpass $CMD > gpurun_out/r2_ncu_full.log 2>&1
echo "full capture rc=$?"

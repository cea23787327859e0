# Round-2d full GPU pass on the current tree: parity suite, smoke, default bench, 20-sweep
# bench, launch list of a short bench (with the small configs), full ncu captures of the X
# passes (one sweep) and of the persistent small-problem kernel at C2 and C4.  Every ncu
# command runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-r02d}
timeout 2400 python -m pytest tests -q -m gpu -rs -s --durations=10 > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.log 2>&1
tail -1 gpurun_out/${T}_bench20.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.log 2>&1
tail -1 gpurun_out/${T}_bench_ref.log | cut -c1-300
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
CMD2="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation --no-small"
timeout 600 $CMD2 > gpurun_out/${T}_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_i8_kernel \
    -s 12 -c 2 -o gpurun_out/${T}_xpass $CMD2 > gpurun_out/${T}_ncu_xpass.log 2>&1
echo "ncu xpass rc=$?"
for c in C2 C4; do
  timeout 300 python tools/small_probe.py 40 $c > gpurun_out/${T}_small_$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_hals -s 1 -c 1 \
      -o gpurun_out/${T}_small_$c python tools/small_probe.py 40 $c > gpurun_out/${T}_ncu_small_$c.log 2>&1
  echo "ncu small $c rc=$?"
done
ENMF_SMALL_DEBUG=1 timeout 300 python tools/small_probe.py 200 > gpurun_out/${T}_small_timeline.log 2>&1
ENMF_SMALL_FUSED=0 timeout 300 python tools/small_probe.py 200 > gpurun_out/${T}_small_unfused.log 2>&1
grep "rep 1" gpurun_out/${T}_small_timeline.log gpurun_out/${T}_small_unfused.log

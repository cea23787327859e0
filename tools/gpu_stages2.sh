# Staged PBCD with the kprev rule: bitwise tests, k* / sweep times at C5, one full ncu capture
# of a whole-iteration-range tc_pbcd_kernel launch (U block, 4th ascent sweep).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_pbcd_stages.py -q -s > gpurun_out/st2_tests.log 2>&1
grep -E "k\* per|stops seen|passed|failed" gpurun_out/st2_tests.log
timeout 600 python tools/kstar_probe.py > gpurun_out/st2_kstar.log 2>&1; tail -14 gpurun_out/st2_kstar.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pbcd_kernel -s 42 -c 1 \
    -o gpurun_out/st2_pbcd python tools/kstar_probe.py > gpurun_out/st2_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/st2_ncu.log

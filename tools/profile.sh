#!/bin/bash
# Profiling recipe (/opt/skills/guides/B200_PROFILING.md) for the bench command; run on a GPU box:
#   gpurun -- 'bash tools/profile.sh'
# 1) plain run of the exact command (must exit 0 before ncu runs it)
# 2) launch list with per-kernel device time (cold-cache, serialised: compare SHARES)
# 3) `--set full` captures (one launch each) of the X-pass kernels, the tensor-core PBCD and HALS
set -u
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py"
$CMD > $OUT/prof_plain.log 2>&1 || { echo "plain run failed"; tail -20 $OUT/prof_plain.log; exit 1; }
tail -1 $OUT/prof_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
SHORT="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"tc_i8_kernel" -s 18 -c 2 \
    -o $OUT/prof_tc $SHORT > $OUT/ncu_full.log 2>&1
echo "full tc rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"tc_pbcd_kernel" -s 2 -c 1 \
    -o $OUT/prof_rows $SHORT > $OUT/ncu_full_rows.log 2>&1
echo "full pbcd rc=$?"
# tc_hals_kernel: launches before the HALS stage return at once; the 27th is an active U block
ncu --set full --clock-control none --import-source on -k regex:"tc_hals_kernel" -s 26 -c 1 \
    -o $OUT/prof_hals python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_full_hals.log 2>&1
echo "full hals rc=$?"

mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "tc_contractions or one_hals_sweep or fullsize" 2>&1 | tail -3 > gpurun_out/xp_tests.log
ENMF_TC_PAIR=1 timeout 900 python -m pytest tests -q -m gpu -x -k "tc_contractions or fullsize" 2>&1 | tail -3 >> gpurun_out/xp_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_i8" --csv --log-file gpurun_out/xp1.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ENMF_TC_PAIR=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_i8" --csv --log-file gpurun_out/xp2.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cat gpurun_out/xp_tests.log

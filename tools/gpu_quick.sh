# Quick GPU check: a pytest selection ($1), a short bench and its launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "$1" 2>&1 | tail -5 > gpurun_out/quick_tests.log
timeout 300 python bench.py --steps ${2:-30} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bq.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python bench.py --steps ${2:-30} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_ncu.log 2>&1
cat gpurun_out/quick_tests.log; tail -1 gpurun_out/bq.log | cut -c1-400

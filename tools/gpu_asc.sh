mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "ascent" -x 2>&1 | tail -5 > gpurun_out/asc.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pbcd" --csv --log-file gpurun_out/pbcd_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1
cat gpurun_out/asc.log

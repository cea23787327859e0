# Staged tensor-core PBCD: bitwise test, ascent parity, k* / sweep times at C5, bench.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_pbcd_stages.py -q -s -x > gpurun_out/st_tests.log 2>&1
tail -12 gpurun_out/st_tests.log
timeout 600 python tools/kstar_probe.py > gpurun_out/st_kstar.log 2>&1; cat gpurun_out/st_kstar.log | tail -15
ENMF_PBCD_STAGES=0 timeout 600 python tools/kstar_probe.py > gpurun_out/st_kstar0.log 2>&1; tail -15 gpurun_out/st_kstar0.log
timeout 1200 python -m pytest tests -q -m gpu -x -k "ascent or smoke or fullsize or multirank" > gpurun_out/st_tests2.log 2>&1
tail -4 gpurun_out/st_tests2.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-ablation --no-small > gpurun_out/st_bench.log 2>&1
tail -1 gpurun_out/st_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print(d['value'], c['stage_rates'], {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, d['e2e']['value'], d['clocks'])"

# tc Gram test, default bench (with C6 in small_configs), NVTX per-sweep launch list at C5.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-r3}
timeout 600 python -m pytest tests/test_gpu_tc_gram.py -q -s > gpurun_out/${T}_tests.log 2>&1; grep -E "tc Gram|passed|failed|Error" gpurun_out/${T}_tests.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print(d['value'], d['e2e']['value'], c['stage_rates'], d['clocks']['sm_mhz'])
print(json.dumps(c['small_configs'].get('C6-reuters-like (CSR)'), indent=0))"
timeout 600 python tools/sweep_launches.py > gpurun_out/${T}_sweeps_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "ascent/" --nvtx-include "hals/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/${T}_sweep_launches.csv python tools/sweep_launches.py \
    > gpurun_out/${T}_ncu_sweeps.log 2>&1
echo "sweep launch list rc=$?"

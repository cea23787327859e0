# Ablation variants on the tensor cores: parity tests, default bench (ablation table).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-abl}
timeout 1800 python -m pytest tests -q -m gpu -x -s -k "ablation or stages or fused or (ascent and tc) or project or smoke" > gpurun_out/${T}_tests.log 2>&1
grep -E "PGD sweep|fixed-step|passed|failed|Error" gpurun_out/${T}_tests.log | head -30
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print(d['value'], d['e2e']['value'], c['stage_rates'], d['clocks']['sm_mhz'])
print(json.dumps(c['ablation_post_rotation'], indent=1))"

# Default bench, the launch list of a short bench (ncu, cold-cache serialised: shares) and
# a full capture of a whole-range tc_pbcd_kernel launch (U block, 3rd ascent sweep).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-bp}
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -1 gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print(d['value'], c['stage_rates'], {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, d['e2e']['value'], d['clocks'])"
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation --no-small"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pbcd_kernel -s 32 -c 1 \
    -o gpurun_out/${T}_pbcd python tools/kstar_probe.py > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"

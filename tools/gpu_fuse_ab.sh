# A/B of the fused U-block HALS through bench.py (default 100-sweep schedule), alternated.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for i in 1 2 3; do
  for f in 1 0; do
    ENMF_FUSE_HALS=$f timeout 600 python bench.py --no-small --no-ablation --no-cpu-baseline --no-e2e > gpurun_out/fab_${f}_${i}.log 2>&1
    echo "fuse=$f $(tail -1 gpurun_out/fab_${f}_${i}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(round(d["value"],2), c["stage_rates"], {k: round(v["ms"],3) for k,v in d["roofline"]["passes"].items()}, d["clocks"]["sm_mhz"])')"
  done
done

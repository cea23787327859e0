# Round-2 profiling pass: bench with C1-C4 / eNMC rates, the cta_group::2 A/B, and one full ncu
# capture of each X pass (the plain command exits 0 first).
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/p2_bench20.log 2>&1
tail -1 gpurun_out/p2_bench20.log | cut -c1-200
for pair in 0 1 0 1; do
  ENMF_TC_PAIR=$pair timeout 600 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation --no-small > gpurun_out/p2_pair$pair.log 2>&1
  echo "pair=$pair $(tail -1 gpurun_out/p2_pair$pair.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], {k: round(v["ms"],3) for k,v in d["roofline"]["passes"].items()}, d["clocks"]["sm_mhz"])')"
done
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-ablation --no-small"
timeout 600 $CMD > gpurun_out/p2_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_i8_kernel \
    -s 12 -c 2 -o gpurun_out/p2_xpass $CMD > gpurun_out/p2_ncu_full.log 2>&1
echo "full capture rc=$?"

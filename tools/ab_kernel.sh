# A/B of one kernel's launch times: ab_old/ (previous build) vs the current tree, alternating.
# usage: bash tools/ab_kernel.sh <kernel-regex> [bench args]
K=$1; shift
ARGS=${@:-"--steps 4 --warmup 3 --no-cpu-baseline --no-e2e"}
mkdir -p gpurun_out; : > gpurun_out/ab_kernel.log
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then b=ab_old/bench.py; else b=bench.py; fi
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv \
      --log-file gpurun_out/ab_$v.csv python $b $ARGS > /dev/null 2>&1
    echo "$v $(python tools/launch_summary.py gpurun_out/ab_$v.csv | head -2 | tr -s ' ' | cut -c1-150 | tr '\n' '|')" >> gpurun_out/ab_kernel.log
  done
done
cat gpurun_out/ab_kernel.log

# A/B of the tensor-core ascent parity: committed tree (ab_prev/) vs working tree.
set -u
mkdir -p gpurun_out
for d in ab_prev .; do
  (cd $d && PYTHONPATH=$PWD timeout 900 python -m pytest tests/test_gpu_shadow.py -q -s -k "ascent and tc" 2>&1 | grep -E "prec=|passed|failed") 
done > gpurun_out/abp.log 2>&1
cat gpurun_out/abp.log

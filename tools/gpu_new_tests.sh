# GPU tests touched in this session + the bench on the one-rank NCCL path.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-nt}
timeout 1200 python -m pytest tests/test_gpu_nccl_single.py tests/test_gpu_heavy_tail.py tests/test_gpu_sparse.py tests/test_gpu_multirank.py -q -rs -s > gpurun_out/${T}_tests.log 2>&1
tail -15 gpurun_out/${T}_tests.log
NCCL_DEBUG=WARN timeout 600 python bench.py --steps 20 --warmup 3 --nccl-single --no-cpu-baseline --no-ablation --no-small > gpurun_out/${T}_bench_nccl1.log 2>&1
tail -1 gpurun_out/${T}_bench_nccl1.log | cut -c1-400

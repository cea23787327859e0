# Fused U-block HALS behind the X V pass: bitwise tests, timing probe, HALS/stage tests.
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
T=${TAG:-fu}
timeout 900 python -m pytest tests/test_gpu_fused_hals.py -q -s -x > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 900 python tools/fuse_probe.py > gpurun_out/${T}_probe.log 2>&1; tail -6 gpurun_out/${T}_probe.log
timeout 1500 python -m pytest tests -q -m gpu -x -k "hals or trajectory or fullsize or smoke or multirank or sparse or final or stages" > gpurun_out/${T}_tests2.log 2>&1
tail -3 gpurun_out/${T}_tests2.log

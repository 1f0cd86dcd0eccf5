set -x
mkdir -p gpurun_out
timeout 300 python tools/configs.py 3 > gpurun_out/r2d_cfg3.jsonl 2> gpurun_out/r2d_cfg3.err
timeout 600 python -m pytest tests/test_gpu_converged.py tests/test_gpu_fast.py tests/test_gpu_pdhg.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2d_tests.log 2>&1; echo rc $? >> gpurun_out/r2d_tests.log
timeout 300 python tools/probe.py 512x256 512x1024 4096x1 > gpurun_out/r2d_probe_exact.log 2>&1
W1MG_FAST=1 timeout 300 python tools/probe.py 512x256 512x1024 4096x1 > gpurun_out/r2d_probe_fast.log 2>&1
true

set -x
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_property.py -x -q -p no:cacheprovider > gpurun_out/pytest_iter.log 2>&1; echo pytest $? >> gpurun_out/pytest_iter.log
timeout 300 python tools/probe.py 4096x1 512x256 256x1024 128x1024 > gpurun_out/probe.log 2>&1
ENGINES=6 timeout 300 python tools/probe.py 4096x1 512x256 256x1024 128x1024 512x1 > gpurun_out/probe3.log 2>&1
true

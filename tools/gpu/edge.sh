timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_rn.py tests/test_gpu_cp.py -x -q -p no:cacheprovider > gpurun_out/pytest_edge.log 2>&1; echo pytest $? >> gpurun_out/pytest_edge.log
true

timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_ml.py tests/test_gpu_property.py -x -q -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest $? >> gpurun_out/pytest_cl.log
timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair.log 2>&1
timeout 300 python tools/configs.py 1 2 > gpurun_out/cfg12.log 2>&1
true

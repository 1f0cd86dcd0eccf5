set -x
timeout 900 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider > gpurun_out/pytest_pdhg.log 2>&1; echo pytest $? >> gpurun_out/pytest_pdhg.log
timeout 300 python tools/configs.py 3 > gpurun_out/cfg3.log 2>&1
W1MG_PDHG_SMALL=2 timeout 300 python tools/configs.py 3 >> gpurun_out/cfg3.log 2>&1
W1MG_PDHG_SMALL=0 timeout 300 python tools/configs.py 3 >> gpurun_out/cfg3.log 2>&1
true

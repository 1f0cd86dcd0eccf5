set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider -k "(fixed_iterations and (rowres or auto)) or config3" > gpurun_out/rs10_tests.log 2>&1; echo rc $? >> gpurun_out/rs10_tests.log
W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 256 > gpurun_out/rs10_probe.log 2>&1
timeout 300 python tools/configs.py 3 > gpurun_out/rs10_cfg3.log 2>&1
true

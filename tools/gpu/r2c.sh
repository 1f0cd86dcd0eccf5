set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2c_pdhg.log 2>&1; echo rc $? >> gpurun_out/r2c_pdhg.log
timeout 300 python tools/configs.py 3 > gpurun_out/r2c_cfg3.jsonl 2> gpurun_out/r2c_cfg3.err
timeout 600 python -m pytest tests/test_gpu_converged.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2c_conv.log 2>&1; echo rc $? >> gpurun_out/r2c_conv.log
true

set -x
mkdir -p gpurun_out
./tools/micro/dmma > gpurun_out/dmma.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider -k "tiny or finest or (fixed_iterations and (rowres or auto)) or config3" > gpurun_out/rs6_tests.log 2>&1; echo rc $? >> gpurun_out/rs6_tests.log
W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 32 64 128 256 512 > gpurun_out/rs6_probe.log 2>&1
timeout 300 python tools/configs.py 3 > gpurun_out/rs6_cfg3.log 2>&1
true

set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider -k "finest or config3" > gpurun_out/rs8_tests.log 2>&1; echo rc $? >> gpurun_out/rs8_tests.log
W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 512 > gpurun_out/rs8_probe.log 2>&1
timeout 300 python tools/configs.py 3 > gpurun_out/rs8_cfg3.log 2>&1
W1MG_PDHG_RS=4 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs8_launches_cfg3.csv python tools/configs.py 3 > gpurun_out/rs8_cfg3_ncu.log 2>&1
true

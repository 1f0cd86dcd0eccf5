set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider -k "finest or (fixed_iterations and (rowres or auto))" > gpurun_out/rs4_tests.log 2>&1; echo rc $? >> gpurun_out/rs4_tests.log
W1MG_PDHG_RS=3 W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 256 512 > gpurun_out/rs4_probe_rs3.log 2>&1
W1MG_PDHG_RS=3 timeout 300 python tools/configs.py 3 > gpurun_out/rs4_cfg3_rs3.log 2>&1
W1MG_PDHG_RS=1 timeout 300 python tools/configs.py 3 > gpurun_out/rs4_cfg3_rs1.log 2>&1
true

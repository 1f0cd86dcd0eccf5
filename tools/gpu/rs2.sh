set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider -k "rowres or auto" > gpurun_out/rs2_tests.log 2>&1; echo rc $? >> gpurun_out/rs2_tests.log
for rs in 3; do
W1MG_PDHG_RS=$rs W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 32 64 128 256 512 > gpurun_out/rs2_probe_rs$rs.log 2>&1
done
W1MG_PDHG_RS=3 timeout 300 python tools/configs.py 3 > gpurun_out/rs2_cfg3_rs3.log 2>&1
W1MG_FAST=1 ENGINES=6 timeout 200 python tools/probe.py 512x1024 4096x1 > gpurun_out/rs2_cp_probe.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_fast.py -x -q -p no:cacheprovider > gpurun_out/rs2_cp_tests.log 2>&1; echo rc $? >> gpurun_out/rs2_cp_tests.log
true

set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_small_cases.py tests/test_studies.py tests/test_gpu_fast.py tests/test_cli.py -q -p no:cacheprovider > gpurun_out/r2q_tests.log 2>&1; echo rc $? >> gpurun_out/r2q_tests.log
W1MG_FAST=1 ENGINES=6 timeout 300 python tools/probe.py 512x256 512x1024 > gpurun_out/r2q_occ5.jsonl 2>&1
W1MG_FAST=1 W1MG_OCC3=6 ENGINES=6 timeout 300 python tools/probe.py 512x256 512x1024 > gpurun_out/r2q_occ6.jsonl 2>&1
true

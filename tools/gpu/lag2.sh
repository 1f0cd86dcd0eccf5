set -x
mkdir -p gpurun_out
W1MG_FAST=1 ENGINES=6 timeout 120 python tools/probe.py 512x1024 256x1024 4096x1 > gpurun_out/lag2_occ5.jsonl 2>&1
W1MG_FAST=1 W1MG_OCC3=4 ENGINES=6 timeout 120 python tools/probe.py 512x1024 256x1024 4096x1 > gpurun_out/lag2_occ4.jsonl 2>&1
ENGINES=6 timeout 120 python tools/probe.py 512x1024 > gpurun_out/lag2_exact.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_headline.py tests/test_gpu_fast.py -x -q -p no:cacheprovider -k "three_sweep or odd_stop or fixed_iterations or headline or fast or batched" > gpurun_out/lag2_tests.log 2>&1; echo rc $? >> gpurun_out/lag2_tests.log
true

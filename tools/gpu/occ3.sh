set -x
mkdir -p gpurun_out
W1MG_FAST=1 ENGINES=6 timeout 200 python tools/probe.py 512x1024 256x1024 4096x1 > gpurun_out/occ5.jsonl 2>&1
W1MG_FAST=1 W1MG_OCC3=4 ENGINES=6 timeout 200 python tools/probe.py 512x1024 256x1024 4096x1 > gpurun_out/occ4.jsonl 2>&1
true

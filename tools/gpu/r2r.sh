set -x
mkdir -p gpurun_out
W1MG_FAST=1 ENGINES=5,6 timeout 600 python tools/probe.py 256x1024 128x1024 256x256 256x1 512x1 384x1 > gpurun_out/r2r_eng.jsonl 2>&1
true

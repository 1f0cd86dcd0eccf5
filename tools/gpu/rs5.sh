set -x
mkdir -p gpurun_out
W1MG_PDHG_RS=3 W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 256 512 > gpurun_out/rs5_probe.log 2>&1
true

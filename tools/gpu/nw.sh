timeout 120 python tools/single_pair_profile.py > gpurun_out/nw.log 2>&1
for nw in 4 8; do echo "== nw $nw" >> gpurun_out/nw.log; W1MG_TMAP_NW=$nw timeout 300 python tools/probe.py 4096x1 2048x1 1024x1 512x1 >> gpurun_out/nw.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_cp.py -q -x -p no:cacheprovider -k "two_sweep or full_size or engine" >> gpurun_out/nw.log 2>&1
true

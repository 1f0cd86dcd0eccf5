ENGINES=3,6 timeout 600 python tools/probe.py 4096x1 2048x1 1024x1 512x256 256x1024 128x1024 512x1 256x1 > gpurun_out/probe3.log 2>&1
timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair.log 2>&1
W1MG_SWEEP=tma3 timeout 300 python tools/single_pair_profile.py >> gpurun_out/single_pair.log 2>&1
true

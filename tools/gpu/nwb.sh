for nw in 4 2 8; do echo "== nw $nw" >> gpurun_out/nwb.log; W1MG_TMAP_NW=$nw timeout 300 python tools/probe.py 512x256 256x1024 4096x1 >> gpurun_out/nwb.log 2>&1; done
true

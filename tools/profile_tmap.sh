#!/bin/bash
# Full ncu capture of the default two-sweep kernel (tensor-map ring) on the
# config-4 finest level (256 pairs x 512^2) and on one 4096^2 grid.
mkdir -p gpurun_out
ENGINES=3 python tools/probe.py 512x256 > gpurun_out/probe_512x256.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cp_sweep2_tmap -s 20 -c 1 \
      -o gpurun_out/prof_tmap_512x256 env ENGINES=3 python tools/probe.py 512x256 > gpurun_out/ncu_full.log 2>&1
ENGINES=3 python tools/probe.py 4096x1 > gpurun_out/probe_4096.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cp_sweep2_tmap -s 20 -c 1 \
      -o gpurun_out/prof_tmap_4096 python tools/probe.py 4096x1 > gpurun_out/ncu_full4096.log 2>&1
echo "profile rc=$?"

ENGINES=6 python tools/probe.py 512x256 > gpurun_out/probe3_512x256.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_sweep3_tmap -s 20 -c 1 \
      -o gpurun_out/prof_tmap3_512x256 env ENGINES=6 python tools/probe.py 512x256 > gpurun_out/ncu3.log 2>&1
true

timeout 600 ncu --set full --clock-control none --import-source on -k regex:pdhg_small -c 1 -o gpurun_out/prof_pdhg_small python tools/configs.py 3 > gpurun_out/pdhg_ncu.log 2>&1
true

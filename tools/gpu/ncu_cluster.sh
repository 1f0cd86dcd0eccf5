timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_cluster -c 1 -o gpurun_out/prof_cluster_cfg1 python tools/configs.py 1 > gpurun_out/ncu_cluster.log 2>&1
true

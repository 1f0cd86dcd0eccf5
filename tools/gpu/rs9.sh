set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs9_launches_cfg3.csv python tools/configs.py 3 > gpurun_out/rs9_cfg3_ncu.log 2>&1; echo rc $? >> gpurun_out/rs9_cfg3_ncu.log
timeout 300 python tools/configs.py 3 > gpurun_out/rs9_cfg3.log 2>&1
true

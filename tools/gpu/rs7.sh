# launch lists (config 3 cascade, one bench step) and ncu summary of the rspf kernel
set -x
mkdir -p gpurun_out
timeout 300 python tools/configs.py 3 > gpurun_out/rs7_cfg3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs7_launches_cfg3.csv python tools/configs.py 3 > gpurun_out/rs7_cfg3_ncu.log 2>&1
PAIRS=2 NCU_TIMEOUT=900 bash tools/launch_list.sh > gpurun_out/rs7_launch_list.log 2>&1
true

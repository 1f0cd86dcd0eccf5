# complete ncu launch list of one timed bench step (2 pairs), long cap
PAIRS=2 NCU_TIMEOUT=2700 bash tools/launch_list.sh > gpurun_out/launch_list_full.log 2>&1
true

#!/bin/bash
# ncu launch list of exactly one timed bench step (bench.py brackets its timed
# region with cudaProfilerStart/Stop).  Plain run first (same command), then
# ncu with --profile-from-start off.  Output: gpurun_out/launches_step.csv
CMD="python bench.py --pairs ${PAIRS:-4} --steps 1 --warmup 3 --no-cpu --no-e2e --no-exact-leg"
mkdir -p gpurun_out
$CMD > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && \
timeout ${NCU_TIMEOUT:-1500} ncu --profile-from-start off --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/launches_step.csv $CMD \
    > gpurun_out/launch_ncu.log 2>&1
echo "ncu rc=$?"

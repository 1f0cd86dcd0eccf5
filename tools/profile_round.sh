#!/bin/bash
# One profiling pass on the GPU box: bench line, launch list, full capture of
# the dominant kernel.  Output under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --pairs 16 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv \
      python bench.py --pairs 16 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/probe.py 512x256 > gpurun_out/probe_512x256.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cp_sweep_tma -s 20 -c 1 \
      -o gpurun_out/prof_tma_512x256 python tools/probe.py 512x256 > gpurun_out/ncu_full.log 2>&1
python tools/probe.py 4096x1 > gpurun_out/probe_4096.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cp_sweep_tma -s 20 -c 1 \
      -o gpurun_out/prof_tma_4096 python tools/probe.py 4096x1 > gpurun_out/ncu_full4096.log 2>&1
echo done

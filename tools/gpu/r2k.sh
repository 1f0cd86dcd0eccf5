# round-2 measurement: bench (both arms), configs 1-5, launch list of one
# timed step, ncu --set full of the dominant kernel (fast numerics)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/r2k_smi.txt
timeout 1500 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2k_bench_ref.json 2> gpurun_out/r2k_bench_ref.err
timeout 900 python tools/configs.py 1 2 3 5 > gpurun_out/r2k_configs.jsonl 2> gpurun_out/r2k_configs.err
W1MG_FAST=1 timeout 300 python tools/probe.py 512x256 512x1024 4096x1 > gpurun_out/r2k_probe_fast.jsonl 2>&1
W1MG_FAST=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_sweep3_tmap -s 20 -c 1 \
    -o gpurun_out/r2k_cp3_fast_512x256 -f env ENGINES=6 W1MG_FAST=1 python tools/probe.py 512x256 > gpurun_out/r2k_ncu3.log 2>&1
NCU_TIMEOUT=900 bash tools/launch_list.sh > gpurun_out/r2k_launch_list.log 2>&1
true

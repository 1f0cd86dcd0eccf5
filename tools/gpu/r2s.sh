set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider > gpurun_out/r2s_fast.log 2>&1; echo rc $? >> gpurun_out/r2s_fast.log
CMD="python bench.py --pairs 1024 --steps 1 --warmup 3 --no-cpu --no-e2e --no-exact-leg"
timeout 900 $CMD > gpurun_out/r2s_default.json 2> gpurun_out/r2s_default.err
W1MG_RESIDENT=2 timeout 900 $CMD > gpurun_out/r2s_res2.json 2> gpurun_out/r2s_res2.err
true

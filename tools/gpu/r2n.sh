set -x
mkdir -p gpurun_out
W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 64 128 256 512 > gpurun_out/r2n_stamps.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pdhg.py tests/test_gpu_converged.py -x -q -p no:cacheprovider > gpurun_out/r2n_tests.log 2>&1; echo rc $? >> gpurun_out/r2n_tests.log
timeout 300 python tools/configs.py 3 > gpurun_out/r2n_cfg3.jsonl 2> gpurun_out/r2n_cfg3.err
true

set -x
mkdir -p gpurun_out
timeout 300 python tools/configs.py 3 > gpurun_out/r2e_cfg3.jsonl 2> gpurun_out/r2e_cfg3.err
timeout 600 python -m pytest tests/test_gpu_pdhg.py tests/test_gpu_converged.py tests/test_cli.py tests/test_studies.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2e_tests.log 2>&1; echo rc $? >> gpurun_out/r2e_tests.log
timeout 900 python tools/acceptance48.py > gpurun_out/r2e_acc.jsonl 2> gpurun_out/r2e_acc.err
true

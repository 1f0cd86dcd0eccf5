set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2b_headline.log 2>&1; echo rc $? >> gpurun_out/r2b_headline.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_headline.py > gpurun_out/r2b_pytest.log 2>&1; echo pytest $? >> gpurun_out/r2b_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
true

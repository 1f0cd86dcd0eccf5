timeout 900 python -m pytest tests/test_gpu_ml.py tests/test_gpu_property.py -x -q -p no:cacheprovider > gpurun_out/pytest_ab2.log 2>&1; echo pytest $? >> gpurun_out/pytest_ab2.log
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 900 python bench.py --no-cpu > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
true

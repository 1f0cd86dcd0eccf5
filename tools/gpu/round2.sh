# full GPU tests, smoke, bench (both arms)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 1700 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/configs.py 1 2 3 5 > gpurun_out/configs.jsonl 2>&1
true

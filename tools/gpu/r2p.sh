set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2p_pytest.log 2>&1; echo pytest $? >> gpurun_out/r2p_pytest.log
timeout 1500 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
PAIRS=2 NCU_TIMEOUT=1200 bash tools/launch_list.sh > gpurun_out/r2p_launch_list.log 2>&1
true

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair.log 2>&1
timeout 300 python tools/probe.py 4096x1 512x1 512x256 256x1 > gpurun_out/probe.log 2>&1

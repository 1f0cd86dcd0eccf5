set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2a_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke $? >> gpurun_out/r2a_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2a_pytest.log 2>&1; echo pytest $? >> gpurun_out/r2a_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
true

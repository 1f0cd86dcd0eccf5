# round-end style measurement: full GPU tests, smoke, bench (both arms),
# launch list of one step, full ncu capture of the dominant kernel
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest $? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
NCU_TIMEOUT=900 bash tools/launch_list.sh > gpurun_out/launch_list.log 2>&1
bash tools/profile_tmap.sh > gpurun_out/profile_tmap.log 2>&1
true

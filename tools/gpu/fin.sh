set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_pdhg.py tests/test_gpu_converged.py tests/test_studies.py tests/test_host.py -x -q -p no:cacheprovider > gpurun_out/fin_tests.log 2>&1; echo rc $? >> gpurun_out/fin_tests.log
timeout 600 python tools/configs.py 1 2 3 5 > gpurun_out/configs.jsonl 2>&1
W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 32 64 128 256 512 > gpurun_out/rs6_probe.log 2>&1
true

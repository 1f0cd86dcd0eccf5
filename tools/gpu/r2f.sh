set -x
mkdir -p gpurun_out
timeout 300 python tools/pdhg_probe.py 400 64 128 256 512 > gpurun_out/r2f_pdhg_probe.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dct_ -s 9 -c 3 -o gpurun_out/r2f_dct513 -f python tools/pdhg_probe.py 4 512 > gpurun_out/r2f_ncu513.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dct_ -s 9 -c 3 -o gpurun_out/r2f_dct257 -f python tools/pdhg_probe.py 4 256 > gpurun_out/r2f_ncu257.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pdhg.py tests/test_gpu_converged.py tests/test_cli.py tests/test_studies.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2f_tests.log 2>&1; echo rc $? >> gpurun_out/r2f_tests.log
timeout 900 python tools/acceptance48.py > gpurun_out/r2f_acc.jsonl 2> gpurun_out/r2f_acc.err
true

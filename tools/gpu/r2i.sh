set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pdhg.py tests/test_gpu_converged.py tests/test_gpu_small_cases.py -x -q -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo rc $? >> gpurun_out/r2i_tests.log
timeout 300 python tools/pdhg_probe.py 400 64 128 256 512 > gpurun_out/r2i_pdhg_probe.jsonl 2>&1
timeout 300 python tools/configs.py 3 > gpurun_out/r2i_cfg3.jsonl 2> gpurun_out/r2i_cfg3.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dct_ -s 9 -c 3 -o gpurun_out/r2i_dct513 -f python tools/pdhg_probe.py 4 512 > gpurun_out/r2i_ncu513.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dct_ -s 9 -c 3 -o gpurun_out/r2i_dct257 -f python tools/pdhg_probe.py 4 256 > gpurun_out/r2i_ncu257.log 2>&1
true

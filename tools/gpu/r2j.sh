set -x
mkdir -p gpurun_out
timeout 300 python tools/pdhg_probe.py 400 64 128 256 512 > gpurun_out/r2j_pdhg_probe.jsonl 2>&1
timeout 300 python tools/configs.py 3 > gpurun_out/r2j_cfg3.jsonl 2> gpurun_out/r2j_cfg3.err
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=20 > gpurun_out/r2j_pytest.log 2>&1; echo pytest $? >> gpurun_out/r2j_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dct_ -s 9 -c 3 -o gpurun_out/r2j_dct257 -f python tools/pdhg_probe.py 4 256 > gpurun_out/r2j_ncu257.log 2>&1
true

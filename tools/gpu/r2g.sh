set -x
mkdir -p gpurun_out
timeout 300 python tools/pdhg_probe.py 400 64 128 256 512 > gpurun_out/r2g_pdhg_probe.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dct_ -s 9 -c 3 -o gpurun_out/r2g_dct513 -f python tools/pdhg_probe.py 4 512 > gpurun_out/r2g_ncu513.log 2>&1
timeout 300 python tools/configs.py 3 > gpurun_out/r2g_cfg3.jsonl 2> gpurun_out/r2g_cfg3.err
timeout 600 python tools/acceptance48.py a8 > gpurun_out/r2g_acc8.jsonl 2> gpurun_out/r2g_acc8.err
timeout 600 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2g_racecheck.log 2>&1; echo rc $? >> gpurun_out/r2g_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2g_synccheck.log 2>&1; echo rc $? >> gpurun_out/r2g_synccheck.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2g_memcheck.log 2>&1; echo rc $? >> gpurun_out/r2g_memcheck.log
true

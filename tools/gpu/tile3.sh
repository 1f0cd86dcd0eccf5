set -x
timeout 600 python -m pytest tests/test_gpu_tile.py -x -q -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo pytest $? >> gpurun_out/pytest_tile.log
W1MG_TILE_DEBUG=1 timeout 300 python tools/single_pair_profile.py > gpurun_out/tile_dbg.log 2>&1
timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair_tile.log 2>&1
true

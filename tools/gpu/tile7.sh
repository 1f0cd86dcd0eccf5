timeout 900 python -m pytest tests/test_gpu_tile.py -x -q -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo pytest $? >> gpurun_out/pytest_tile.log
W1MG_TILE=1 W1MG_TILE_DEPTH=2 W1MG_TILE_DEBUG=1 timeout 300 python tools/single_pair_profile.py > gpurun_out/tile2_dbg.log 2>&1
echo "== depth2" > gpurun_out/tile_sp.log; W1MG_TILE=1 W1MG_TILE_DEPTH=2 timeout 300 python tools/single_pair_profile.py >> gpurun_out/tile_sp.log 2>&1
echo "== depth2 min32" >> gpurun_out/tile_sp.log; W1MG_TILE=1 W1MG_TILE_DEPTH=2 W1MG_TILE_MIN=32 timeout 300 python tools/single_pair_profile.py >> gpurun_out/tile_sp.log 2>&1
true

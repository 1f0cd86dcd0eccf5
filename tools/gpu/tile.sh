set -x
timeout 600 python -m pytest tests/test_gpu_tile.py -x -q -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo pytest $? >> gpurun_out/pytest_tile.log
timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair_tile.log 2>&1
W1MG_TILE=0 timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair_notile.log 2>&1
for g in 6 8 10; do W1MG_TILE_GRID=$g timeout 300 python tools/single_pair_profile.py >> gpurun_out/single_pair_grid.log 2>&1; done
W1MG_TILE_MIN=32 timeout 300 python tools/single_pair_profile.py >> gpurun_out/single_pair_grid.log 2>&1
true

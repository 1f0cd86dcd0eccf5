set -x
timeout 600 python -m pytest tests/test_gpu_tile.py -x -q -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo pytest $? >> gpurun_out/pytest_tile.log
W1MG_TILE_DEBUG=1 timeout 300 python tools/single_pair_profile.py > gpurun_out/tile_dbg.log 2>&1
W1MG_TILE=0 timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair_notile.log 2>&1
timeout 300 python tools/single_pair_profile.py > gpurun_out/single_pair_tile.log 2>&1
W1MG_TILE_GRID=8 timeout 300 python tools/single_pair_profile.py >> gpurun_out/single_pair_tile.log 2>&1
W1MG_TILE_MIN=32 timeout 300 python tools/single_pair_profile.py >> gpurun_out/single_pair_tile.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_ml.py tests/test_gpu_slab.py tests/test_gpu_property.py -x -q -p no:cacheprovider > gpurun_out/pytest_iter.log 2>&1; echo pytest $? >> gpurun_out/pytest_iter.log
true

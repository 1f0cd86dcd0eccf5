set -x
timeout 900 python -m pytest tests/test_gpu_tile.py -x -q -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo pytest $? >> gpurun_out/pytest_tile.log
echo "== default" > gpurun_out/tile_sp.log; timeout 300 python tools/single_pair_profile.py >> gpurun_out/tile_sp.log 2>&1
for cfg in "W1MG_TILE=1 W1MG_TILE_DEPTH=2" "W1MG_TILE=1 W1MG_TILE_DEPTH=2 W1MG_TILE_GRID=10" "W1MG_TILE=1 W1MG_TILE_DEPTH=2 W1MG_TILE_MIN=32" "W1MG_TILE=1 W1MG_TILE_DEPTH=2 W1MG_TILE_GRID=8 W1MG_TILE_MIN=32"; do
  echo "== $cfg" >> gpurun_out/tile_sp.log; env $cfg timeout 300 python tools/single_pair_profile.py >> gpurun_out/tile_sp.log 2>&1; done
true

W1MG_TILE_DEBUG=1 timeout 300 python tools/single_pair_profile.py > gpurun_out/tile_dbg.log 2>&1
W1MG_TILE_DEBUG=1 W1MG_TILE_GRID=6 timeout 300 python tools/single_pair_profile.py > gpurun_out/tile_dbg6.log 2>&1
true

W1MG_TILE=1 W1MG_TILE_DEPTH=2 W1MG_TILE_DEBUG=1 timeout 300 python tools/single_pair_profile.py > gpurun_out/tile2_dbg.log 2>&1
true

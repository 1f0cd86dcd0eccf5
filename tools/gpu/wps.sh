for cfg in "" "W1MG_WARPS_PER_SM=8" "W1MG_WARPS_PER_SM=4" "W1MG_WARPS_PER_SM=8 W1MG_TMAP_NW=4" "W1MG_WARPS_PER_SM=12"; do
  echo "== $cfg" >> gpurun_out/wps.log; env $cfg timeout 120 python tools/single_pair_profile.py >> gpurun_out/wps.log 2>&1; done
true

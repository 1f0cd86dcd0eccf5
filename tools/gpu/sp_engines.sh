# one-pair cascade level times under engine / geometry switches
for cfg in "" "W1MG_SWEEP=tma" "W1MG_SWEEP=ldg" "W1MG_WARPS_PER_SM=16" "W1MG_WARPS_PER_SM=64" "W1MG_WARPS_PER_SM=128" "W1MG_PDL=0" "W1MG_TMAP_NW=2" "W1MG_TMAP_NW=8"; do
  echo "== $cfg" >> gpurun_out/sp_engines.log
  env $cfg timeout 120 python tools/single_pair_profile.py >> gpurun_out/sp_engines.log 2>&1
done
true

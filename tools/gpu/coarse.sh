# one-pair coarse levels under the resident-engine switches
for cfg in "" "W1MG_RESIDENT=2" "W1MG_CLUSTER_PICK=0" "W1MG_RESIDENT=3" "W1MG_TILE=2 W1MG_TILE_MIN=32"; do
  echo "== $cfg" >> gpurun_out/coarse.log
  env $cfg timeout 120 python tools/single_pair_profile.py >> gpurun_out/coarse.log 2>&1
done
true

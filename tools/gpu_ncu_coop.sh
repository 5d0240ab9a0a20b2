#!/bin/bash
# ncu --set full of one cooperative GMRES launch (cfg5 level 1 FC phase), tools only
mkdir -p gpurun_out
for c in ${CFGS:-cfg5}; do
  MGRIT_COOP_RW=${RW:-0} timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:gmres2d_coop -s ${SKIP:-0} -c 1 -o gpurun_out/${c}_coop -f python tools/profile_phase.py $c L1_FC_corrected > gpurun_out/ncu_${c}_coop.log 2>&1
  echo "$c coop rc=$?"
done

#!/bin/bash
# ncu --set full captures (one launch each) of the cfg5 fine SL step kernel and
# the cfg5 level-1 cooperative GMRES kernel, from one eager V-cycle.
mkdir -p gpurun_out
TAG=${TAG:-r02}
for k in ${KERNELS:-sl2d_strip gmres2d_coop}; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$k -c 1 -o gpurun_out/${TAG}_cfg5_$k -f python tools/profile_iteration.py cfg5 \
    > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done

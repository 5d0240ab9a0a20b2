#!/bin/bash
# ncu --set full of the 2D SL step (cfg4 p=3 512-wide, cfg5 p=5 1024-wide) and
# the cooperative 2D GMRES (cfg4 level 1) on the final kernels (tools only)
mkdir -p gpurun_out
TAG=${TAG:-r01f}
for c in cfg4 cfg5; do
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:sl2d_kernel -c 1 -o gpurun_out/${TAG}_${c}_sl2d -f python tools/profile_iteration.py $c > gpurun_out/ncu_sl2d_$c.log 2>&1
echo "$c sl2d rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:gmres2d_coop --launch-skip 5 -c 1 -o gpurun_out/${TAG}_cfg4_gmres2d -f python tools/profile_iteration.py cfg4 > gpurun_out/ncu_g2d.log 2>&1
echo "g2d rc=$?"

#!/bin/bash
# ncu --set full capture of the 2D SL step kernel (cfg4 p=3, cfg5 p=5), tools only
mkdir -p gpurun_out
for c in ${CFGS:-cfg4 cfg5}; do
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:sl2d_kernel -c 1 -o gpurun_out/${c}_sl2d -f python tools/profile_iteration.py $c > gpurun_out/ncu_sl2d_$c.log 2>&1
echo "$c sl2d rc=$?"
done

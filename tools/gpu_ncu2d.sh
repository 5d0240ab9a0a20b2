#!/bin/bash
# ncu --set full captures of the 2D kernels (tools only)
export MGRIT_COOP_ROWS=${MGRIT_COOP_ROWS:--1}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:gmres2d_coop --launch-skip 5 -c 1 -o gpurun_out/cfg4_gmres2d -f python tools/profile_iteration.py cfg4 > gpurun_out/ncu_g2d.log 2>&1
echo "g2d rc=$?"
if [ -n "$SL2D" ]; then
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:sl2d_kernel -c 1 -o gpurun_out/cfg5_sl2d -f python tools/profile_iteration.py cfg5 > gpurun_out/ncu_sl2d.log 2>&1
echo "sl2d rc=$?"
fi

#!/bin/bash
# ncu --set full of the fine 2D SL step: separable-table kernel vs column-strip kernel (tools only)
mkdir -p gpurun_out
for c in ${CFGS:-cfg5}; do
  for v in ${VARIANTS:-sep strip}; do
    if [ $v = sep ]; then export MGRIT_SL2D_SEP_ROWS=${SEPROWS:-16}; K=sl2d_sep_kernel; else export MGRIT_SL2D_SEP_ROWS=0; K=sl2d_strip_kernel; fi
    timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:$K -c 1 -o gpurun_out/${c}_${v} -f python tools/profile_iteration.py $c > gpurun_out/ncu_${c}_${v}.log 2>&1
    echo "$c $v rc=$?"
  done
done

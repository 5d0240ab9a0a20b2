#!/bin/bash
# DRAM bytes of whole fused phases (every launch of the phase, cold cache) for
# the bench lines' roofline `traffic` fields (tools only; run under gpurun).
mkdir -p gpurun_out
for spec in ${SPECS:-cfg1:L0_FC_fine cfg1_085h:L0_FC_fine cfg3:L1_F_RES_corrected cfg4:L0_FC_fine cfg4:L1_F_RES_corrected cfg5:L0_FC_fine cfg5:L0_F_RES_fine}; do
  c=${spec%%:*}; k=${spec#*:}
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/traffic_${c}_${k}.csv python tools/profile_phase.py $c $k \
    > gpurun_out/traffic_${c}_${k}.log 2>&1
  echo "$c $k rc=$?"
done

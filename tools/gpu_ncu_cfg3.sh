#!/bin/bash
# ncu --set full of the cfg3 fine-level FC phase (tools only)
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:phase_kernel -c 1 -o gpurun_out/cfg3_L0_FC -f python tools/profile_iteration.py cfg3 > gpurun_out/ncu_cfg3.log 2>&1
echo "cfg3 rc=$?"

#!/bin/bash
# cfg2 bench launch list + ncu --set full captures of the fine SL phase and the
# top coarse phase (tools only; run under gpurun, one GPU).  TAG names the files.
TAG=${TAG:-r01e}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
# fine-level FC phase (first phase_kernel launch of one profiled iteration)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:phase_kernel -c 1 -o gpurun_out/${TAG}_L0_FC_fine -f python tools/profile_iteration.py cfg2 > gpurun_out/ncu_l0.log 2>&1
echo "l0 rc=$?"
# top coarse phase: L4 F_RES (6th cluster phase launch: L2 FC, L2 F_RES, L3 FC, L3 F_RES, L4 FC, L4 F_RES)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:cl_phase_kernel --launch-skip 5 -c 1 -o gpurun_out/${TAG}_L4_F_RES -f python tools/profile_iteration.py cfg2 > gpurun_out/ncu_l4.log 2>&1
echo "l4 rc=$?"
# level-1 phase on two CTAs per SM (first phase_kernel launch with 256 threads)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base mangled -k regex:"phase_kernelILi3ELi1ELi256ELi16ELb1ELi2E" -c 1 -o gpurun_out/${TAG}_L1_FC -f python tools/profile_iteration.py cfg2 > gpurun_out/ncu_l1.log 2>&1
echo "l1 rc=$?"

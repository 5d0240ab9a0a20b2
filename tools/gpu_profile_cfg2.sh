#!/bin/bash
# launch list + ncu --set full captures for the cfg2 bench (tools only; run under gpurun)
set -x
mkdir -p gpurun_out
for v in mgs mgs_lowsync; do for pol in auto cta cluster; do
  timeout 300 python bench.py --no-cpu --no-e2e --gmres-variant $v --launch-policy $pol > gpurun_out/bv_cfg2_${v}_${pol}.json 2>&1
  echo "$v $pol rc=$?"
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
# fine-level FC phase (first phase_kernel launch of one profiled iteration)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:phase_kernel -c 1 -o gpurun_out/L0_FC_fine -f python tools/profile_iteration.py cfg2 > gpurun_out/ncu_l0.log 2>&1
echo "l0 rc=$?"
# top coarse kernel: the cluster phase kernel (first launch = L1 FC)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:cl_phase_kernel -c 1 -o gpurun_out/cl_phase -f python tools/profile_iteration.py cfg2 > gpurun_out/ncu_cl.log 2>&1
echo "cl rc=$?"

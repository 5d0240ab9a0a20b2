#!/bin/bash
# FP64 thread-instruction counts + DRAM bytes of the column-strip 2D SL kernel
# (one fine F-step launch of cfg4 and cfg5), for profiles/ncu_fp64.json
for c in cfg4 cfg5; do
  timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --profile-from-start off -k regex:sl2d_strip -c 1 --csv --log-file gpurun_out/fp64_strip_$c.csv \
    python tools/profile_iteration.py $c > /dev/null 2>&1; echo "$c rc=$?"
done

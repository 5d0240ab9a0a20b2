#!/bin/bash
# bench the 1D configs with both GMRES variants (tools only)
for c in cfg1 cfg1_085h cfg2 cfg3; do for v in mgs mgs_lowsync; do
python bench.py --config $c --no-cpu --no-e2e --gmres-variant $v > gpurun_out/bv_${c}_${v}.json 2>&1
done; done

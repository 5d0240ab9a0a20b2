#!/bin/bash
# bench cfg2 under every launch policy x GMRES variant (tools only)
for pol in cta cluster auto; do for v in mgs mgs_lowsync; do
python bench.py --no-cpu --no-e2e --launch-policy $pol --gmres-variant $v > gpurun_out/b_${pol}_${v}.json 2>gpurun_out/b_${pol}_${v}.err
done; done

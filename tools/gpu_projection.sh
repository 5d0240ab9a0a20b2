#!/bin/bash
# time-sharded engine on one GPU: bit-identity tests, then the per-rank V-cycle projections (tools/project_scaling.py)
set -u
mkdir -p gpurun_out
python -m pytest tests/test_timepar_gpu.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_timepar.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_timepar.log
for c in ${CFGS:-cfg5 cfg4 cfg3 cfg2}; do
  timeout 900 python tools/project_scaling.py $c > gpurun_out/${TAG:-r02e}_scaling_projection_$c.json 2> gpurun_out/proj_$c.err; echo "$c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/${TAG:-r02e}_scaling_projection_$c.json')); print('$c', {k: (v['projected_ms_per_iteration'], v.get('projected_speedup_vs_P1')) for k,v in d['per_P'].items()})"
done

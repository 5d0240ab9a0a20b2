#!/bin/bash
python -m pytest tests/test_gpu_production2d.py tests/test_gpu_parity.py -m gpu -q -k "corrected or 2d or sl2d" -p no:cacheprovider > gpurun_out/pytest_r02f.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_r02f.log
python tools/sensitivity_probe.py cfg3 7 > gpurun_out/sens_cfg3.json 2> gpurun_out/sens_cfg3.err; echo sens=$?
for v in mgs mgs_lowsync; do
  python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu --no-e2e --gmres-variant $v > gpurun_out/b5_$v.json 2> gpurun_out/b5_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/b5_$v.json').read().strip().splitlines()[-1]); b=d['kernel_breakdown_ms']
print('$v', round(d['ms_per_step'],1), d['solve']['iterations'], {k: round(x,2) for k,x in b.items()})"
done

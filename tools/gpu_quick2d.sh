#!/bin/bash
# 2D parity subset + cfg5/cfg4 bench lines (tools only)
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sl2d_sep.py tests/test_gpu_parity.py tests/test_gpu_production2d.py tests/test_timepar_gpu.py -m gpu -q -k "2d or sl2d or sep or fine_fc or fullsize or fused or corrected" -p no:cacheprovider > gpurun_out/pytest_quick2d.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_quick2d.log
for cfg in ${CFGS:-cfg5 cfg4}; do
  python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/quick_${cfg}.json 2> gpurun_out/quick_${cfg}.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/quick_{sys.argv[1]}.json").read().strip().splitlines()[-1])
b = d["kernel_breakdown_ms"]
print(sys.argv[1], "ms/solve %.1f" % d["ms_per_step"], "iters", d["solve"]["iterations"],
      {k: round(v, 2) for k, v in b.items()}, "sl", d["sl_step_roofline"]["frac"], d["parity"].get("max_history_dev_over_r0"), flush=True)
PY
done

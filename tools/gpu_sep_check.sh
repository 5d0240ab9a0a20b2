#!/bin/bash
# Separable 2D SL kernel: parity tests, then the strip-height sweep on cfg5/cfg4
# (MGRIT_SL2D_SEP_ROWS = 0 (column-strip kernel), 8, 16, 32, 64, unset = auto).
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sl2d_sep.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_sep.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_sep.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_production2d.py -m gpu -q -k "2d or sl2d" -p no:cacheprovider > gpurun_out/pytest_sep2.log 2>&1; echo pytest2=$?; tail -3 gpurun_out/pytest_sep2.log
for cfg in cfg5 cfg4; do
  for nb in ${ROWS:-0 8 16 32 auto}; do
    if [ $nb = auto ]; then unset MGRIT_SL2D_SEP_ROWS; else export MGRIT_SL2D_SEP_ROWS=$nb; fi
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e \
      > gpurun_out/sep_${cfg}_${nb}.json 2> gpurun_out/sep_${cfg}_${nb}.err
    python - "$cfg" "$nb" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/sep_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
b = d["kernel_breakdown_ms"]
print(sys.argv[1], "sep rows", sys.argv[2], "ms/solve %.1f" % d["ms_per_step"], "iters", d["solve"]["iterations"],
      "L0_FC %.3f" % b["L0_FC_fine"], "L0_F_RES %.3f" % b["L0_F_RES_fine"], "L0_INJ_F %.3f" % b["L0_INJ_F_fine"],
      "seq %.2f" % d["sequential_gpu_ms"], "hbm frac", d["sl_step_roofline"]["frac"], flush=True)
PY
  done
done

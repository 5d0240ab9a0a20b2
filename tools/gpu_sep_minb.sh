#!/bin/bash
# sl2d_sep_kernel occupancy sweep (MGRIT_SL2D_SEP_MINB = resident CTAs per SM the kernel is compiled for)
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sl2d_sep.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_sep.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_sep.log
for cfg in cfg5 cfg4; do
  for mb in ${MINBS:-2 3 4}; do
   for nb in ${ROWS:-32}; do
    MGRIT_SL2D_SEP_ROWS=$nb MGRIT_SL2D_SEP_MINB=$mb python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e \
      > gpurun_out/sepmb_${cfg}_${mb}_${nb}.json 2> gpurun_out/sepmb_${cfg}_${mb}_${nb}.err
    python - "$cfg" "$mb" "$nb" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/sepmb_{sys.argv[1]}_{sys.argv[2]}_{sys.argv[3]}.json").read().strip().splitlines()[-1])
b = d["kernel_breakdown_ms"]
print(sys.argv[1], "minb", sys.argv[2], "rows", sys.argv[3], "ms/solve %.1f" % d["ms_per_step"], "iters", d["solve"]["iterations"],
      "L0_FC %.3f" % b["L0_FC_fine"], "L0_F_RES %.3f" % b["L0_F_RES_fine"], "L0_INJ_F %.3f" % b["L0_INJ_F_fine"],
      "seq %.2f" % d["sequential_gpu_ms"], "hbm frac", d["sl_step_roofline"]["frac"], flush=True)
PY
   done
  done
done

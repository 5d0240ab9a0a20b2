#!/bin/bash
# SL-step strip-height sweep (MGRIT_SL2D_STRIP = 0 (per-node kernel), 2, 4, 8)
# on configs 4 and 5: solve time + the fine FC phase from bench.py's breakdown.
set -u
mkdir -p gpurun_out
for cfg in cfg5 cfg4; do
  for nb in 0 2 4 8; do
    MGRIT_SL2D_STRIP=$nb python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e \
      > gpurun_out/strip_${cfg}_${nb}.json 2> gpurun_out/strip_${cfg}_${nb}.err
    python - "$cfg" "$nb" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/strip_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
b = d["kernel_breakdown_ms"]
print(sys.argv[1], "strip", sys.argv[2], "ms/solve %.1f" % d["ms_per_step"], "iters", d["solve"]["iterations"],
      "L0_FC %.3f" % b["L0_FC_fine"], "L0_F_RES %.3f" % b["L0_F_RES_fine"], "L0_INJ_F %.3f" % b["L0_INJ_F_fine"],
      "fp64 frac", d["sl_step_roofline"]["fp64"]["frac"], flush=True)
PY
  done
done

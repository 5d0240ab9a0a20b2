#!/bin/bash
# cooperative GMRES: systems in flight (MGRIT_COOP_ROWS) x on-chip w (MGRIT_COOP_RW) on cfg5 / cfg4
set -u
mkdir -p gpurun_out
for cfg in ${CFGS:-cfg5}; do
  for rows in ${ROWSS:-1 2 3}; do
   for rw in ${RWS:-0 1}; do
    MGRIT_COOP_ROWS=$rows MGRIT_COOP_RW=$rw python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e \
      > gpurun_out/rows_${cfg}_${rows}_${rw}.json 2> gpurun_out/rows_${cfg}_${rows}_${rw}.err
    python - "$cfg" "$rows" "$rw" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/rows_{sys.argv[1]}_{sys.argv[2]}_{sys.argv[3]}.json").read().strip().splitlines()[-1])
b = d["kernel_breakdown_ms"]
print(sys.argv[1], "rows", sys.argv[2], "rw", sys.argv[3], "ms/solve %.1f" % d["ms_per_step"], "iters", d["solve"]["iterations"],
      {k: round(v, 2) for k, v in b.items() if "corrected" in k}, flush=True)
PY
   done
  done
done

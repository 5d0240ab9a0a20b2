"""Per-phase V-cycle times of a 1D bench config under one kernel shape for
the corrected levels (measurement input of the cluster-size policy,
step1d_cl.cu cl_wave_cost100):
    python tools/cluster_sizes.py cfg2 cluster2     (or cta, cluster4/8/16, auto)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402

name, policy = sys.argv[1], sys.argv[2]
P.set_launch_policy(policy)
cfg = P.SolverConfig(**bench.CONFIGS[name])
levels = P.build_hierarchy(cfg)
rep, _ = P.solve(cfg, levels, output="device")
bd, _ = bench.kernel_breakdown(levels, cfg)
out = {"config": name, "policy": policy,
       "iterations": rep.iterations, "history_last": float(rep.residual_norms[-1]),
       "chains": {f"L{i}": lv.n_steps // lv.cf for i, lv in enumerate(levels[:-1])},
       "ms": {k: round(v["ms_total"], 4) for k, v in bd.items()}}
print(json.dumps(out))

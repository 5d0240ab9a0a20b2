"""Rounding sensitivity of a full-size solve: the same config solved with
kernel shapes / GMRES variants whose reductions sum in different orders
(all equally valid restatements of the reference's BLAS inner products).
Their spread is the floor any two implementations can agree to; the
deviation from the reference fixture is printed beside it.

    python tools/sensitivity_probe.py cfg3 [max_iters] > gpurun_out/sens_cfg3.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402

name = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else None
kw = dict(bench.CONFIGS[name])
if k is not None:
    kw.update(max_iters=k, rtol=0.0)
fx = bench._load_fixture(bench.FULLSIZE.get(name, "")) if name in bench.FULLSIZE else None
variants = [("auto", "mgs"), ("cta", "mgs"), ("auto", "mgs_lowsync")]
if kw.get("dim", 1) == 2:
    variants = [("auto", "mgs"), ("auto", "mgs_lowsync")]
out = {"config": name, "runs": {}}
hists, cols = {}, {}
idx = None
if fx is not None:
    idx = torch.as_tensor(fx["cols_idx"], device="cuda")
for policy, variant in variants:
    P.set_launch_policy(policy)
    cfg = P.SolverConfig(**kw, gmres_variant=variant)
    levels = P.build_hierarchy(cfg)
    rep, U = P.solve(cfg, levels, output="device")
    key = f"{policy}/{variant}"
    hists[key] = np.asarray(rep.residual_norms)
    if idx is not None:
        cols[key] = U[:, idx].cpu().numpy()
    out["runs"][key] = {"iterations": rep.iterations, "status": rep.status}
    del U, levels
    torch.cuda.empty_cache()
keys = list(hists)
r0 = hists[keys[0]][0]


def dev(a, b):
    m = min(len(a), len(b))
    return float(np.max(np.abs(a[:m] - b[:m])) / r0)


out["history_spread_over_r0"] = {f"{a} vs {b}": dev(hists[a], hists[b]) for i, a in enumerate(keys)
                                 for b in keys[i + 1:]}
if fx is not None:
    out["history_dev_vs_fixture_over_r0"] = {kk: dev(h, fx["hist"]) for kk, h in hists.items()}
    j = min(len(fx["hist"]), min(len(h) for h in hists.values())) - 1
    if j >= 1 and k is not None and k <= len(fx["cols"]):
        ref = fx["cols"][k - 1]
        out["iterate_cols_rel_vs_fixture"] = {kk: float(np.linalg.norm(c - ref) / np.linalg.norm(ref))
                                              for kk, c in cols.items()}
        out["iterate_cols_rel_spread"] = {
            f"{a} vs {b}": float(np.linalg.norm(cols[a] - cols[b]) / np.linalg.norm(ref))
            for i, a in enumerate(keys) for b in keys[i + 1:]}
print(json.dumps(out))

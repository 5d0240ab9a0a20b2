"""Round-2 kernels under compute-sanitizer: the separable 2D SL kernel (every
strip height, both wraps, the per-node fallback of large-CFL levels, all
output forms through a short solve) and the cluster-split plain-SL sweep.
    compute-sanitizer --tool memcheck python tools/sanitize_r02.py
    compute-sanitizer --tool racecheck python tools/sanitize_r02.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_13382_b200 as P  # noqa: E402

for nb in ("8", "16", "32"):
    os.environ["MGRIT_SL2D_SEP_ROWS"] = nb
    for p in (1, 3, 5):
        cfg = P.SolverConfig(n_x=256, n_t=16, dim=2, wave_speed="B4", p=p, schedule=4, seed=3, u0="sin4", max_iters=2)
        rep, U = P.solve(cfg)
        assert np.isfinite(U).all()
        print("sep rows", nb, "p", p, rep.iterations, rep.status)
os.environ.pop("MGRIT_SL2D_SEP_ROWS")
# large-CFL plain-SL coarse levels: staged tiles that do not fit fall back per node
cfg = P.SolverConfig(n_x=256, n_t=64, dim=2, wave_speed="B4", p=3, schedule=4, seed=3, u0="sin4",
                     operator_kind="rediscretized", departure_policy="erk_rediscretized", max_iters=1)
rep, U = P.solve(cfg)
print("rediscretized", rep.iterations, rep.status)
# cluster-split plain-SL sweep
for pol, n_x, p in (("cluster2", 1024, 1), ("cluster8", 4096, 3), ("cluster16", 4096, 5), ("cluster16", 16384, 5)):
    prev = P.set_launch_policy(pol)
    cfg = P.SolverConfig(n_x=n_x, n_t=16, wave_speed="B2", p=p, schedule=4)
    U = P.sequential_reference(cfg, P.build_hierarchy(cfg), output="device")
    P.set_launch_policy(prev)
    assert torch.isfinite(U).all()
    print(pol, n_x, p, "ok")
print("ok")

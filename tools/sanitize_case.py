"""Small 1D + 2D solves (all phase kinds) for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_13382_b200 as P  # noqa: E402

for kw in (dict(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4),
           dict(n_x=4096, n_t=64, wave_speed="B2", p=3, schedule=4),
           dict(n_x=64, n_t=64, wave_speed="C2", p=1, schedule=4, relaxation="F"),
           dict(n_x=64, n_t=128, wave_speed="C1", p=1, schedule=8, max_levels=2),
           dict(n_x=16, n_t=64, dim=2, wave_speed="C5", p=3, schedule=4),
           dict(n_x=32, n_t=64, dim=2, wave_speed="B4", p=5, schedule=4, operator_kind="forward_euler",
                max_levels=2)):
    cfg = P.SolverConfig(**kw, max_iters=3)
    rep, U = P.solve(cfg)
    print(kw, rep.iterations, rep.status)
print("ok")
